# cfg3: tile size x concurrent-remote hot warps
mkdir -p gpurun_out/r2o
O=gpurun_out/r2o
for v in "256 8" "256 7" "256 9" "128 8" "128 6" "512 8" "512 10"; do
  set -- $v
  KUR_CONC_REMOTE=$2 python bench.py --config 3 --steps 50 --warmup 5 --no-cpu --no-e2e --tile-rows $1 > $O/x.json 2> $O/x.err || { echo fail; tail -3 $O/x.err; continue; }
  python -c "import json; d=json.load(open('$O/x.json')); r=d['roofline']; print('cfg3 tile $1 hot_warps $2', round(d['value'],1), 'ms/step', round(d['ms_per_step'],4), 'stage_us', round(1000*r['avg_launch_ms'],2))"
done
