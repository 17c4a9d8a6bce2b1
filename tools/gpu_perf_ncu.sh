# perf cycle: parity subset, bench cfg5/4/3, one ncu --set full of k_stage on cfg5
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_methods.py -x -q -m gpu > gpurun_out/pytest_gpu.log 2>&1; echo pytest=$?
tail -2 gpurun_out/pytest_gpu.log
bash tools/gpu_perf.sh 5 4 3
ncu --set full --clock-control none --import-source on -k regex:k_stage -s 6 -c 1 -o gpurun_out/prof5 python bench.py --steps 2 --warmup 3 --no-cpu --no-e2e > gpurun_out/ncu_f5.log 2>&1; echo ncu=$?
