# quick GPU cycle: parity tests + config 5 and 4 bench lines
mkdir -p gpurun_out
timeout 900 python -m pytest tests -x -q -m gpu > gpurun_out/pytest_gpu.log 2>&1; echo pytest=$?
tail -3 gpurun_out/pytest_gpu.log
python bench.py --steps 20 --warmup 3 --no-cpu > gpurun_out/b5.json 2> gpurun_out/b5.err; echo b5=$?
python bench.py --config 4 --steps 50 --warmup 3 --no-cpu --no-e2e > gpurun_out/b4.json 2> gpurun_out/b4.err; echo b4=$?
python bench.py --config 3 --steps 50 --warmup 3 --no-cpu --no-e2e > gpurun_out/b3.json 2> gpurun_out/b3.err; echo b3=$?
for c in 5 4 3; do python -c "
import json; d=json.load(open('gpurun_out/b$c.json')); r=d['roofline']; print('cfg$c', round(d['value'],1), 'RHS/s stage_ms', round(r['avg_launch_ms'],4), 'frac', round(r['frac'],3), 'tiles', d['plan']['n_tiles'], d['plan']['rows_per_tile'], 'build_s', round(d['host']['build_s'],1))"; done
tail -3 gpurun_out/b5.err
