# persistent kernel (counter barrier), pooled row pieces (cfg3/cfg4 padding), full GPU suite, bench lines
mkdir -p gpurun_out/r2d
O=gpurun_out/r2d
for c in 2 3 4; do
  python bench.py --config $c --steps 50 --warmup 5 --no-cpu > $O/cfg$c.json 2> $O/cfg$c.err; echo cfg$c rc=$?
  python -c "import json; d=json.load(open('$O/cfg$c.json')); r=d['roofline']; print('cfg$c', round(d['value'],1), 'stage_us', round(1000*r['avg_launch_ms'],2), 'frac', round(r['frac'],3), 'e2e', round(d['e2e']['value'],1), 'launches', d['gpu_launches'])"
done
timeout 2400 python -m pytest tests -x -q -m gpu > $O/pytest_gpu.log 2>&1; echo pytest=$?; tail -2 $O/pytest_gpu.log
python bench.py --steps 20 --warmup 5 > $O/bench_default.json 2> $O/bench_default.err; echo default rc=$?
python -c "import json; d=json.load(open('$O/bench_default.json')); r=d['roofline']; print('cfg5', round(d['value'],1), 'stage_us', round(1000*r['avg_launch_ms'],2), 'frac', round(r['frac'],3), 'e2e', round(d['e2e']['value'],1), 'cpu', d['cpu_baseline']['value'], d['clocks'])"
ncu --set full --clock-control none --import-source on -k regex:k_persist -c 1 -o $O/cfg2_persist python bench.py --config 2 --steps 3 --warmup 3 --no-cpu --no-e2e > $O/ncu_f2.log 2>&1; echo full2=$?
ncu --set full --clock-control none --import-source on -k regex:k_stage -s 6 -c 1 -o $O/cfg4_stage python bench.py --config 4 --steps 2 --warmup 3 --no-cpu --no-e2e > $O/ncu_f4.log 2>&1; echo full4=$?
