# full GPU suite + smoke at the final commit
mkdir -p gpurun_out/r2fin2
O=gpurun_out/r2fin2
timeout 2700 python -m pytest tests -q -m gpu > $O/pytest_gpu.log 2>&1; echo pytest=$?; tail -2 $O/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo smoke=$?; tail -1 $O/smoke.log
python bench.py --config 3 --steps 50 --warmup 5 --no-cpu --no-e2e > $O/bench_cfg3.json 2> $O/bench_cfg3.err; echo cfg3=$?
python -c "import json; d=json.load(open('$O/bench_cfg3.json')); r=d['roofline']; print('cfg3', round(d['value'],1), 'stage_us', round(1000*r['avg_launch_ms'],2), 'tiles', d['plan']['n_tiles'])"
