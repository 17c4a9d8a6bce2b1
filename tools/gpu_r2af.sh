# remote pass vs inline (concurrent) remote part on configs 3 and 4, current build
mkdir -p gpurun_out/r2af
O=gpurun_out/r2af
for r in 1 2; do for rp in auto on; do for c in 3 4; do
  st=20; [ $c = 3 ] && st=100
  python bench.py --config $c --steps $st --warmup 5 --no-cpu --no-e2e --remote-pass $rp > $O/x.json 2> $O/x.err || { echo fail; tail -3 $O/x.err; continue; }
  python -c "import json; d=json.load(open('$O/x.json')); r=d['roofline']; print('round $r remote_pass $rp cfg$c', round(d['value'],1), 'stage_us', round(1000*r['avg_launch_ms'],2), 'k_remote_us', round(1000*r['k_remote_ms'],2))"
done; done; done
