# final bench lines of the last build (deferred S4 record) + launch list cfg3, smoke
mkdir -p gpurun_out/r2fin4
O=gpurun_out/r2fin4
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo smoke=$?; tail -1 $O/smoke.log
python bench.py --steps 20 --warmup 5 > $O/bench_default.json 2> $O/bench_default.err; echo default=$?
python -c "import json; d=json.load(open('$O/bench_default.json')); r=d['roofline']; print('cfg5', round(d['value'],1), 'stage_us', round(1000*r['avg_launch_ms'],2), 'frac', round(r['frac'],3), 'e2e', round(d['e2e']['value'],1), 'cpu', d['cpu_baseline']['value'], d['clocks'])"
for c in 1 2 3 4; do
  python bench.py --config $c --steps 50 --warmup 5 > $O/bench_cfg$c.json 2> $O/bench_cfg$c.err; echo cfg$c=$?
  python -c "import json; d=json.load(open('$O/bench_cfg$c.json')); r=d['roofline']; print('cfg$c', round(d['value'],1), 'ms/step', round(d['ms_per_step'],5), 'stage_us', round(1000*r['avg_launch_ms'],2), 'frac', round(r['frac'],3), 'e2e', round(d['e2e']['value'],1), 'launches', d['gpu_launches'])"
done
python bench.py --impl reference --steps 2 --warmup 3 > $O/bench_reference.json 2> $O/bench_reference.err; echo reference=$?
CMD="python bench.py --config 3 --steps 3 --warmup 3 --no-cpu --no-e2e"
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches_cfg3.csv $CMD > $O/ncu_l3.log 2>&1; echo launches3=$?
python tools/launch_summary.py $O/launches_cfg3.csv > $O/launches_cfg3_summary.txt 2>&1
CMD="python bench.py --config 5 --steps 3 --warmup 3 --no-cpu --no-e2e"
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches_cfg5.csv $CMD > $O/ncu_l5.log 2>&1; echo launches5=$?
python tools/launch_summary.py $O/launches_cfg5.csv > $O/launches_cfg5_summary.txt 2>&1
