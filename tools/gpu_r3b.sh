# same-box A/B: persist grid barrier with (A = libkur_a.so, the committed
# default build) vs acquire polls, A) vs two fewer block barriers per local_reduce (B); config 2, 4 rounds;
# then the persist tests under B
mkdir -p gpurun_out
for r in 1 2 3 4; do for v in a b; do
  L=paper_2102_07167_b200/libkur_$v.so
  KUR_LIB=$L python bench.py --config 2 --steps 200 --warmup 5 --no-cpu --no-e2e > gpurun_out/ab.json 2> gpurun_out/ab.err || { echo fail $v; tail -3 gpurun_out/ab.err; continue; }
  python -c "
import json; d=json.load(open('gpurun_out/ab.json')); r=d['roofline']; print('round $r cfg2 $v', round(d['value'],1), 'ms/step', round(d['ms_per_step']*1000,2), 'us; stage_us', round(1000*r['avg_launch_ms'],2))"
done; done
KUR_LIB=paper_2102_07167_b200/libkur_b.so timeout 600 python -m pytest tests/test_gpu_persist.py -q -x 2>&1 | tail -3
