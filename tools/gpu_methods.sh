mkdir -p gpurun_out
timeout 1200 python -m pytest tests -x -q -m gpu > gpurun_out/pytest_gpu.log 2>&1; echo pytest=$?
tail -15 gpurun_out/pytest_gpu.log
timeout 600 python tools/crossover.py > gpurun_out/crossover.jsonl 2> gpurun_out/crossover.err; echo crossover=$?
tail -3 gpurun_out/crossover.err
