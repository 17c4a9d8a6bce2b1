mkdir -p gpurun_out/r2e
O=gpurun_out/r2e
python bench.py --steps 20 --warmup 5 > $O/bench_default.json 2> $O/bench_default.err; echo default rc=$?
python -c "import json; d=json.load(open('$O/bench_default.json')); r=d['roofline']; print('cfg5', round(d['value'],1), 'stage_us', round(1000*r['avg_launch_ms'],2), 'frac', round(r['frac'],3), 'e2e', round(d['e2e']['value'],1), 'cpu', d['cpu_baseline']['value'], d['clocks'], d['gpu_launches'])"
python bench.py --config 2 --steps 200 --warmup 5 --no-cpu > $O/cfg2.json 2> $O/cfg2.err; echo cfg2 rc=$?
python -c "import json; d=json.load(open('$O/cfg2.json')); r=d['roofline']; print('cfg2', round(d['value'],1), 'stage_us', round(1000*r['avg_launch_ms'],2), 'e2e', round(d['e2e']['value'],1))"
bash tools/gpu_sweep_cfg3.sh
CMD="python bench.py --config 5 --steps 2 --warmup 3 --no-cpu --no-e2e"
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches_cfg5.csv $CMD > $O/ncu_l5.log 2>&1; echo launches5=$?
ncu --set full --clock-control none --import-source on -k regex:k_stage -s 6 -c 1 -o $O/cfg5_stage $CMD > $O/ncu_f5.log 2>&1; echo full5=$?
ncu --set full --clock-control none --import-source on -k regex:k_remote -s 6 -c 1 -o $O/cfg5_remote $CMD > $O/ncu_r5.log 2>&1; echo full5r=$?
ncu --set full --clock-control none --import-source on -k regex:k_persist -c 1 -o $O/cfg2_persist python bench.py --config 2 --steps 3 --warmup 3 --no-cpu --no-e2e > $O/ncu_f2.log 2>&1; echo full2=$?
