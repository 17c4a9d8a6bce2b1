mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_edge.py -x -q -m gpu -k remainder > gpurun_out/pt_rem.log 2>&1; echo rem=$?; tail -1 gpurun_out/pt_rem.log
bash tools/gpu_sweep2.sh 3 "256 512" "512 1024 2048" "off on"
bash tools/gpu_sweep2.sh 4 "256 512" "2048" "off on"
bash tools/gpu_sweep2.sh 5 "2048" "1024 2048 4096" "on"
