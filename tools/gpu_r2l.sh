mkdir -p gpurun_out/r2l
O=gpurun_out/r2l
timeout 1200 python -m pytest "tests/test_gpu_sharded.py::test_concurrent_inline_remote_bitwise" "tests/test_gpu_sharded.py::test_remote_modes_bitwise" tests/test_gpu_parity.py -k "concurrent or remote_modes or config3 or small or layout" -x -q -m gpu > $O/pytest.log 2>&1; echo pytest=$?; tail -2 $O/pytest.log
for r in 1 2; do for k in 0 4 6 8 10 12; do
  KUR_CONC_REMOTE=$k python bench.py --config 3 --steps 50 --warmup 5 --no-cpu --no-e2e > $O/x.json 2> $O/x.err || { echo fail; tail -3 $O/x.err; }
  python -c "import json; d=json.load(open('$O/x.json')); r=d['roofline']; print('round $r cfg3 conc_remote=$k', round(d['value'],1), 'ms/step', round(d['ms_per_step'],4), 'stage_us', round(1000*r['avg_launch_ms'],2))"
done; done
for k in 0 8; do
  KUR_CONC_REMOTE=$k python bench.py --config 4 --steps 20 --warmup 5 --no-cpu --no-e2e > $O/x.json 2> $O/x.err || { echo fail; tail -3 $O/x.err; }
  python -c "import json; d=json.load(open('$O/x.json')); r=d['roofline']; print('cfg4 conc_remote=$k', round(d['value'],1), 'ms/step', round(d['ms_per_step'],4), 'stage_us', round(1000*r['avg_launch_ms'],2))"
done
