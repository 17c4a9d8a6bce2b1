# cluster-resident stage timing breakdown (KUR_CZ_DBG: 1 skip parts, 2 no DSMEM reads, 4 no part barriers)
mkdir -p gpurun_out/r2z4
O=gpurun_out/r2z4
for r in 1 2; do for dbg in 0 1 2 3 4; do
  KUR_CZ_DBG=$dbg python bench.py --config 3 --steps 100 --warmup 5 --no-cpu --no-e2e > $O/x.json 2> $O/x.err || { echo fail; tail -3 $O/x.err; continue; }
  python -c "import json; d=json.load(open('$O/x.json')); r=d['roofline']; print('round $r dbg $dbg cfg3', round(d['value'],1), 'ms/step', round(d['ms_per_step'],5), 'stage_us', round(1000*r['avg_launch_ms'],2))"
done; done
