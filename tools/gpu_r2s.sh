mkdir -p gpurun_out/r2s
timeout 1500 python tools/scaling_model.py --worlds 2 8 --steps 4 > gpurun_out/r2s/scaling_model.txt 2>&1; echo model=$?; head -6 gpurun_out/r2s/scaling_model.txt
