# k_remote z-gather cache variants (libkur_v1: ld.global.ca, v2: nc L1::evict_first, v3: nc L1::evict_last)
# and the k_remote shared-memory carveout (KUR_REM_CARVEOUT), config 5
mkdir -p gpurun_out/r2ad
O=gpurun_out/r2ad
for r in 1 2; do for v in libkur libkur_v1 libkur_v2 libkur_v3 carve0 carve100; do
  case $v in carve0) L=libkur; E="KUR_REM_CARVEOUT=0";; carve100) L=libkur; E="KUR_REM_CARVEOUT=100";; *) L=$v; E="KUR_X=0";; esac
  env $E KUR_LIB=$PWD/paper_2102_07167_b200/$L.so python bench.py --config 5 --steps 20 --warmup 5 --no-cpu --no-e2e > $O/x.json 2> $O/x.err || { echo fail $v; tail -3 $O/x.err; continue; }
  python -c "import json; d=json.load(open('$O/x.json')); r=d['roofline']; print('round $r $v cfg5', round(d['value'],1), 'stage_us', round(1000*r['avg_launch_ms'],2), 'k_remote_us', round(1000*r['k_remote_ms'],2))"
done; done
