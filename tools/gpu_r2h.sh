# PDL between stage kernels + batched finish loads: A/B (KUR_NO_PDL=1) on cfg3/4/5, parity subset
mkdir -p gpurun_out/r2h
O=gpurun_out/r2h
timeout 1500 python -m pytest tests/test_gpu_parity.py tests/test_gpu_edge.py tests/test_gpu_persist.py tests/test_gpu_methods.py -x -q -m gpu > $O/pytest.log 2>&1; echo pytest=$?; tail -2 $O/pytest.log
for r in 1 2; do for c in 3 4 5; do for p in 0 1; do
  if [ $p = 1 ]; then export KUR_NO_PDL=1; fi
  python bench.py --config $c --steps 20 --warmup 5 --no-cpu --no-e2e > $O/x.json 2> $O/x.err || { echo fail; tail -3 $O/x.err; }
  unset KUR_NO_PDL
  python -c "import json; d=json.load(open('$O/x.json')); r=d['roofline']; print('round $r cfg$c nopdl=$p', round(d['value'],1), 'ms/step', round(d['ms_per_step'],4), 'stage_us', round(1000*r['avg_launch_ms'],2))"
done; done; done
