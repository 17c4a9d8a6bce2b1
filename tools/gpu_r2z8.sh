# cluster-resident stage: 512 vs 1024 threads per CTA vs the tile plan (cfg3), CZ tests at 1024
mkdir -p gpurun_out/r2z8
O=gpurun_out/r2z8
for r in 1 2; do for v in tile cz512 cz1024; do
  case $v in tile) E="KUR_CZ=0";; cz512) E="KUR_CZ_THREADS=512";; cz1024) E="KUR_CZ_THREADS=1024";; esac
  env $E python bench.py --config 3 --steps 100 --warmup 5 --no-cpu --no-e2e > $O/x.json 2> $O/x.err || { echo fail; tail -3 $O/x.err; continue; }
  python -c "import json; d=json.load(open('$O/x.json')); r=d['roofline']; print('round $r $v cfg3', round(d['value'],1), 'ms/step', round(d['ms_per_step'],5), 'stage_us', round(1000*r['avg_launch_ms'],2))"
done; done
KUR_CZ_THREADS=1024 timeout 600 python -m pytest tests/test_gpu_cluster.py -x -q -m gpu > $O/pytest_cz.log 2>&1; echo pytest_cz1024=$?; tail -3 $O/pytest_cz.log
