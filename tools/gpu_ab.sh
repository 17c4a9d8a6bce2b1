# same-box A/B of two builds: libkur_a.so (A) vs libkur.so (B); bash tools/gpu_ab.sh "<configs>" [rounds]
mkdir -p gpurun_out
for r in $(seq ${2:-2}); do for c in $1; do for v in a b; do
  L=paper_2102_07167_b200/libkur.so; [ $v = a ] && L=paper_2102_07167_b200/libkur_a.so
  KUR_LIB=$L python bench.py --config $c --steps 20 --warmup 3 --no-cpu --no-e2e > gpurun_out/ab.json 2> gpurun_out/ab.err || { echo fail $v $c; tail -3 gpurun_out/ab.err; continue; }
  python -c "
import json; d=json.load(open('gpurun_out/ab.json')); r=d['roofline']; print('round $r cfg$c $v', round(d['value'],1), 'stage_us', round(1000*r['avg_launch_ms'],2), 'k_stage_us', round(1000*(r.get('k_stage_ms') or 0),2))"
done; done; done
