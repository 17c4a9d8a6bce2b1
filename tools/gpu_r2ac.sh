# random z gathers with / without L1 allocation (libkur_na.so = -DKUR_Z_NOALLOC): cfg5 (k_remote), cfg3/cfg4 (inline)
mkdir -p gpurun_out/r2ac
O=gpurun_out/r2ac
for r in 1 2; do for lib in libkur libkur_na; do for c in 5 3 4; do
  st=20; [ $c = 3 ] && st=100
  KUR_LIB=$PWD/paper_2102_07167_b200/$lib.so python bench.py --config $c --steps $st --warmup 5 --no-cpu --no-e2e > $O/x.json 2> $O/x.err || { echo fail; tail -3 $O/x.err; continue; }
  python -c "import json; d=json.load(open('$O/x.json')); r=d['roofline']; print('round $r $lib cfg$c', round(d['value'],1), 'stage_us', round(1000*r['avg_launch_ms'],2), 'k_remote_us', round(1000*r['k_remote_ms'],2))"
done; done; done
