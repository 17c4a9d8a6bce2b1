mkdir -p gpurun_out/r2x
O=gpurun_out/r2x
for r in 1 2; do for tr in 0 1824 1664; do
  python bench.py --config 5 --steps 20 --warmup 5 --no-cpu --no-e2e --tile-rows $tr > $O/x.json 2> $O/x.err || { echo fail; tail -3 $O/x.err; continue; }
  python -c "import json; d=json.load(open('$O/x.json')); r=d['roofline']; print('round $r cfg5 tile $tr', round(d['value'],1), 'ms/step', round(d['ms_per_step'],4), 'stage_us', round(1000*r['avg_launch_ms'],2), 'tiles', d['plan']['n_tiles'])"
done; done
for tr in 1824 1664; do
timeout 1500 python tools/scaling_model.py --worlds 8 --steps 4 --tile-rows $tr > $O/scaling_model_$tr.txt 2>&1; grep "^G=" $O/scaling_model_$tr.txt
done
