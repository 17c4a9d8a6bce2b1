mkdir -p gpurun_out/r2u
O=gpurun_out/r2u
timeout 2400 python -m pytest tests/test_gpu_sharded.py tests/test_gpu_adaptive.py tests/test_gpu_methods.py -q -m gpu > $O/pytest.log 2>&1; echo pytest=$?; tail -2 $O/pytest.log
timeout 1500 python tools/scaling_model.py --worlds 2 4 8 --steps 4 --remote-pass on > $O/scaling_model_pass.txt 2>&1; echo model=$?; grep "^G=" $O/scaling_model_pass.txt
timeout 1500 python tools/scaling_model.py --worlds 8 --steps 4 > $O/scaling_model_auto.txt 2>&1; grep "^G=" $O/scaling_model_auto.txt
