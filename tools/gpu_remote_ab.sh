# remote-part modes A/B (KUR_REMOTE_MODE 0 = k_remote pass, 1 = in-kernel warp + TMA gathers,
# 2 = in-kernel warp + LDG gathers): parity subset under each mode, then cfg5 stage times
mkdir -p gpurun_out
for m in 1 2; do
  KUR_REMOTE_MODE=$m timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_edge.py tests/test_gpu_sharded.py -x -q -m gpu > gpurun_out/pytest_rm$m.log 2>&1; echo mode$m pytest=$?; tail -1 gpurun_out/pytest_rm$m.log
done
for r in 1 2; do for c in ${CFGS:-5}; do for m in 0 1 2; do
  KUR_REMOTE_MODE=$m python bench.py --config $c --steps 20 --warmup 3 --no-cpu --no-e2e --remote-pass ${RP:-auto} > gpurun_out/ab.json 2> gpurun_out/ab.err || { echo fail $m $c; tail -3 gpurun_out/ab.err; continue; }
  python -c "
import json; d=json.load(open('gpurun_out/ab.json')); r=d['roofline']; print('round $r cfg$c mode$m', round(d['value'],1), 'stage_us', round(1000*r['avg_launch_ms'],2), 'k_stage_us', round(1000*(r.get('k_stage_ms') or 0),2), 'k_remote_us', round(1000*(r.get('k_remote_ms') or 0),2))"
done; done; done
