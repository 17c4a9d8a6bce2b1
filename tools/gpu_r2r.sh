mkdir -p gpurun_out/r2r
O=gpurun_out/r2r
timeout 900 python -m pytest tests/test_gpu_persist.py -x -q -m gpu > $O/pytest.log 2>&1; echo pytest=$?; tail -1 $O/pytest.log
python bench.py --config 2 --steps 200 --warmup 5 --no-cpu --no-e2e > $O/x.json 2> $O/x.err; python -c "import json; d=json.load(open('$O/x.json')); r=d['roofline']; print('cfg2', round(d['value'],1), 'stage_us', round(1000*r['avg_launch_ms'],3))"
timeout 1500 python tools/scaling_model.py --worlds 2 4 8 --steps 4 > $O/scaling_model.txt 2>&1; echo model=$?; cat $O/scaling_model.txt | head -5
