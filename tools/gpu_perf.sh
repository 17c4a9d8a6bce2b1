# perf-only cycle: configs given as args (default 5 4)
mkdir -p gpurun_out
for c in ${@:-5 4}; do
  python bench.py --config $c --steps 20 --warmup 3 --no-cpu --no-e2e > gpurun_out/p$c.json 2> gpurun_out/p$c.err; echo p$c=$?
  python -c "
import json; d=json.load(open('gpurun_out/p$c.json')); r=d['roofline']; print('cfg$c', round(d['value'],1), 'RHS/s stage_ms', round(r['avg_launch_ms'],4), 'frac', round(r['frac'],3), 'tiles', d['plan']['n_tiles'], d['plan']['rows_per_tile'], 'build_s', round(d['host']['build_s'],1), d['clocks']['sm_mhz'])"
done
