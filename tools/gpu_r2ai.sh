# overlapped remote pass on by default: full GPU suite, same-box A/B cfg3/cfg5 (KUR_REMOTE_OVERLAP=0 vs default)
mkdir -p gpurun_out/r2ai
O=gpurun_out/r2ai
for r in 1 2; do for ov in 0 def; do for c in 5 3; do
  st=20; [ $c = 3 ] && st=100
  if [ $ov = def ]; then E="KUR_X=0"; else E="KUR_REMOTE_OVERLAP=0"; fi
  env $E python bench.py --config $c --steps $st --warmup 5 --no-cpu --no-e2e > $O/x$c$ov.json 2> $O/x.err || { echo fail; tail -3 $O/x.err; continue; }
  python -c "import json; d=json.load(open('$O/x$c$ov.json')); r=d['roofline']; print('round $r overlap $ov cfg$c', round(d['value'],1), 'stage_us', round(1000*r['avg_launch_ms'],2), 'frac', round(r['frac'],3), 'launches', d['gpu_launches'], r.get('remote_overlap') is not None)"
done; done; done
timeout 2700 python -m pytest tests -q -m gpu > $O/pytest_gpu.log 2>&1; echo pytest=$?; tail -2 $O/pytest_gpu.log
