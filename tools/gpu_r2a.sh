# round-2 check: same-box A/B of the round-1 build (a), the new build without the remote-warp
# branch (b) and the new build (c, KUR_REMOTE_MODE=0) on cfg5; then the full GPU suite
mkdir -p gpurun_out
for r in 1 2 3; do for v in a b c; do
  L=paper_2102_07167_b200/libkur.so; [ $v = a ] && L=paper_2102_07167_b200/libkur_a.so; [ $v = b ] && L=paper_2102_07167_b200/libkur_b.so
  KUR_LIB=$L python bench.py --config 5 --steps 20 --warmup 3 --no-cpu --no-e2e > gpurun_out/ab.json 2> gpurun_out/ab.err || { echo fail $v; tail -3 gpurun_out/ab.err; continue; }
  python -c "
import json; d=json.load(open('gpurun_out/ab.json')); r=d['roofline']; print('round $r $v', round(d['value'],1), 'stage_us', round(1000*r['avg_launch_ms'],2), 'k_stage_us', round(1000*(r.get('k_stage_ms') or 0),2), 'k_remote_us', round(1000*(r.get('k_remote_ms') or 0),2), d['clocks']['sm_mhz'])"
done; done
timeout 2400 python -m pytest tests -x -q -m gpu > gpurun_out/pytest_gpu_r2a.log 2>&1; echo pytest=$?; tail -5 gpurun_out/pytest_gpu_r2a.log
