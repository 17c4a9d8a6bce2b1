# k_stage shared-memory carveout (KUR_STAGE_CARVEOUT %): L1 left for the inline remote gathers (configs 3, 4)
mkdir -p gpurun_out/r2ae
O=gpurun_out/r2ae
for r in 1 2; do for cv in none 60 65 72 80 100; do for c in 3 4; do
  st=20; [ $c = 3 ] && st=100
  if [ $cv = none ]; then E="KUR_X=0"; else E="KUR_STAGE_CARVEOUT=$cv"; fi
  env $E python bench.py --config $c --steps $st --warmup 5 --no-cpu --no-e2e > $O/x.json 2> $O/x.err || { echo fail; tail -3 $O/x.err; continue; }
  python -c "import json; d=json.load(open('$O/x.json')); r=d['roofline']; print('round $r carve $cv cfg$c', round(d['value'],1), 'stage_us', round(1000*r['avg_launch_ms'],2))"
done; done; done
