# kernel iteration cycle: parity subset, per-tile phase profile, perf lines (cfg 5 4 3)
mkdir -p gpurun_out
timeout 1500 python -m pytest tests/test_gpu_parity.py tests/test_gpu_sharded.py tests/test_gpu_methods.py tests/test_gpu_next.py tests/test_gpu_adaptive.py -x -q -m gpu > gpurun_out/pytest_gpu.log 2>&1; echo pytest=$?
tail -4 gpurun_out/pytest_gpu.log
for c in 5 4 3; do python tools/tile_profile.py --config $c; done > gpurun_out/tp.log 2>&1; cat gpurun_out/tp.log
bash tools/gpu_perf.sh 5 4 3 2
