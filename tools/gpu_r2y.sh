# deferred block sums (KUR_LAZY_T): GPU suite subset + same-box A/B on configs 3, 4, 5
mkdir -p gpurun_out/r2y
O=gpurun_out/r2y
timeout 1500 python -m pytest tests/test_gpu_parity.py tests/test_gpu_edge.py tests/test_gpu_methods.py tests/test_gpu_next.py tests/test_gpu_host_buffers.py tests/test_gpu_sharded.py tests/test_gpu_adaptive.py -x -q -m gpu > $O/pytest.log 2>&1; echo pytest=$?; tail -3 $O/pytest.log
for r in 1 2; do for lz in 0 1; do for c in 3 4 5; do
  st=20; [ $c = 3 ] && st=100
  KUR_LAZY_T=$lz python bench.py --config $c --steps $st --warmup 5 --no-cpu --no-e2e > $O/x.json 2> $O/x.err || { echo fail; tail -3 $O/x.err; continue; }
  python -c "import json; d=json.load(open('$O/x.json')); r=d['roofline']; print('round $r lazy $lz cfg$c', round(d['value'],1), 'ms/step', round(d['ms_per_step'],5), 'stage_us', round(1000*r['avg_launch_ms'],2))"
done; done; done
