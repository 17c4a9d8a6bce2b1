# persistent kernel with flag publication, L2-keep index policy for small pools
mkdir -p gpurun_out/r2c
O=gpurun_out/r2c
timeout 1200 python -m pytest tests/test_gpu_persist.py tests/test_gpu_parity.py tests/test_gpu_edge.py -x -q -m gpu > $O/pytest.log 2>&1; echo pytest=$?; tail -2 $O/pytest.log
python bench.py --config 2 --steps 200 --warmup 5 --no-cpu > $O/cfg2.json 2> $O/cfg2.err; echo cfg2 rc=$?
python -c "import json; d=json.load(open('$O/cfg2.json')); r=d['roofline']; print('cfg2', round(d['value'],1), 'stage_us', round(1000*r['avg_launch_ms'],2), 'e2e', round(d['e2e']['value'],1))"
for r in 1 2; do for k in 0 1; do
  KUR_L2_KEEP=$k python bench.py --config 3 --steps 50 --warmup 5 --no-cpu --no-e2e > $O/cfg3_k$k.json 2> $O/cfg3_k$k.err
  python -c "import json; d=json.load(open('$O/cfg3_k$k.json')); r=d['roofline']; print('round $r cfg3 l2keep=$k', round(d['value'],1), 'stage_us', round(1000*r['avg_launch_ms'],2))"
done; done
python bench.py --config 5 --steps 20 --warmup 3 --no-cpu --no-e2e > $O/cfg5.json 2> $O/cfg5.err
python -c "import json; d=json.load(open('$O/cfg5.json')); r=d['roofline']; print('cfg5', round(d['value'],1), 'stage_us', round(1000*r['avg_launch_ms'],2), 'k_stage', round(1000*r['k_stage_ms'],2))"
ncu --set full --clock-control none --import-source on -k regex:k_persist -c 1 -o $O/cfg2_persist python bench.py --config 2 --steps 3 --warmup 3 --no-cpu --no-e2e > $O/ncu_f2.log 2>&1; echo full2=$?
KUR_L2_KEEP=1 ncu --set full --clock-control none --import-source on -k regex:k_stage -s 6 -c 1 -o $O/cfg3_stage python bench.py --config 3 --steps 2 --warmup 3 --no-cpu --no-e2e > $O/ncu_f3.log 2>&1; echo full3=$?
