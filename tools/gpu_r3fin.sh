# final-state validation after the acquire-poll grid barrier: full GPU suite, smoke, bench lines for
# every config + reference, ncu full capture of config 2's persistent kernel, launch list config 2
mkdir -p gpurun_out/r3fin
O=gpurun_out/r3fin
timeout 2700 python -m pytest tests -q -m gpu > $O/pytest_gpu.log 2>&1; echo pytest=$?; tail -3 $O/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo smoke=$?; tail -1 $O/smoke.log
python bench.py --steps 20 --warmup 5 > $O/bench_default.json 2> $O/bench_default.err; echo default=$?
python -c "import json; d=json.load(open('$O/bench_default.json')); r=d['roofline']; print('cfg5', round(d['value'],1), 'stage_us', round(1000*r['avg_launch_ms'],2), 'frac', round(r['frac'],3), 'e2e', round(d['e2e']['value'],1), 'cpu', d['cpu_baseline']['value'], d['clocks'])"
for c in 1 2 3 4; do
  python bench.py --config $c --steps 50 --warmup 5 > $O/bench_cfg$c.json 2> $O/bench_cfg$c.err; echo cfg$c=$?
  python -c "import json; d=json.load(open('$O/bench_cfg$c.json')); r=d['roofline']; print('cfg$c', round(d['value'],1), 'ms/step', round(d['ms_per_step'],5), 'stage_us', round(1000*r['avg_launch_ms'],2), 'frac', round(r['frac'],3), 'e2e', round(d['e2e']['value'],1), 'launches', d['gpu_launches'])"
done
python bench.py --impl reference --steps 2 --warmup 3 > $O/bench_reference.json 2> $O/bench_reference.err; echo reference=$?
CMD="python bench.py --config 2 --steps 3 --warmup 3 --no-cpu --no-e2e"
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches_cfg2.csv $CMD > $O/ncu_l2.log 2>&1; echo launches2=$?
python tools/launch_summary.py $O/launches_cfg2.csv > $O/launches_cfg2_summary.txt 2>&1
ncu --set full --clock-control none --import-source on -k regex:k_persist -c 1 -o $O/cfg2_persist $CMD > $O/ncu_f2.log 2>&1; echo full2=$?
