mkdir -p gpurun_out/r2q
O=gpurun_out/r2q
for r in 1 2 3; do for v in r7 r8; do
  L=paper_2102_07167_b200/libkur.so; [ $v = r8 ] && L=paper_2102_07167_b200/libkur_r8.so
  KUR_LIB=$L python bench.py --config 2 --steps 200 --warmup 5 --no-cpu --no-e2e > $O/x.json 2> $O/x.err || { echo fail; tail -3 $O/x.err; }
  python -c "import json; d=json.load(open('$O/x.json')); r=d['roofline']; print('round $r cfg2 $v', round(d['value'],1), 'ms/step', round(d['ms_per_step'],5), 'stage_us', round(1000*r['avg_launch_ms'],3))"
done; done
