# quick A/B: parity subset + perf lines
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_edge.py tests/test_gpu_sharded.py -x -q -m gpu > gpurun_out/pytest_gpu.log 2>&1; echo pytest=$?; tail -1 gpurun_out/pytest_gpu.log
bash tools/gpu_perf.sh ${@:-3 4 5}
