# full evidence cycle: parity tests, smoke, bench lines for every config, cfg5 launch list + one full ncu capture
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -x -q -m gpu > gpurun_out/pytest_gpu.log 2>&1; echo pytest=$?
tail -3 gpurun_out/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo smoke=$?
bash tools/gpu_bench_all.sh
for c in 5 1 2 3 4; do python -c "
import json; d=json.load(open('gpurun_out/b$c.json')); r=d['roofline']; print('cfg$c', round(d['value'],1), 'RHS/s stage_ms', round(r['avg_launch_ms'],4), 'frac', round(r['frac'],3), 'e2e', round(d['e2e']['value'],1) if d['e2e'] else None, d['clocks'])"; done
