mkdir -p gpurun_out/r2v
timeout 1500 python tools/scaling_model.py --worlds 2 4 8 --steps 4 > gpurun_out/r2v/scaling_model.txt 2>&1; echo model=$?; grep "^G=" gpurun_out/r2v/scaling_model.txt
