mkdir -p gpurun_out/r2t
timeout 1500 python tools/scaling_model.py --worlds 4 8 --steps 4 --remote-pass on > gpurun_out/r2t/scaling_model_pass.txt 2>&1; echo model=$?; head -4 gpurun_out/r2t/scaling_model_pass.txt
