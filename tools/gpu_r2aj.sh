# RK4 S4 deferring its reduction + step record to the next S1 (KUR_LAZY_REC=0 vs default): A/B cfg3/cfg4/cfg5, GPU suite
mkdir -p gpurun_out/r2aj
O=gpurun_out/r2aj
for r in 1 2; do for lr in 0 1; do for c in 3 4 5; do
  st=20; [ $c = 3 ] && st=100
  KUR_LAZY_REC=$lr python bench.py --config $c --steps $st --warmup 5 --no-cpu --no-e2e > $O/x.json 2> $O/x.err || { echo fail; tail -3 $O/x.err; continue; }
  python -c "import json; d=json.load(open('$O/x.json')); r=d['roofline']; print('round $r lazy_rec $lr cfg$c', round(d['value'],1), 'stage_us', round(1000*r['avg_launch_ms'],2))"
done; done; done
timeout 2700 python -m pytest tests -q -m gpu > $O/pytest_gpu.log 2>&1; echo pytest=$?; tail -2 $O/pytest_gpu.log
