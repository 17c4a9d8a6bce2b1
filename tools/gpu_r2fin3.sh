# final-state evidence with the overlapped remote pass: bench lines for every config + reference, launch
# lists cfg3/cfg5, ncu full captures of k_stage and k_remote (cfg3, cfg5), smoke
mkdir -p gpurun_out/r2fin3
O=gpurun_out/r2fin3
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo smoke=$?; tail -1 $O/smoke.log
python bench.py --steps 20 --warmup 5 > $O/bench_default.json 2> $O/bench_default.err; echo default=$?
python -c "import json; d=json.load(open('$O/bench_default.json')); r=d['roofline']; print('cfg5', round(d['value'],1), 'stage_us', round(1000*r['avg_launch_ms'],2), 'frac', round(r['frac'],3), 'e2e', round(d['e2e']['value'],1), 'cpu', d['cpu_baseline']['value'], d['clocks'])"
for c in 1 2 3 4; do
  python bench.py --config $c --steps 50 --warmup 5 > $O/bench_cfg$c.json 2> $O/bench_cfg$c.err; echo cfg$c=$?
  python -c "import json; d=json.load(open('$O/bench_cfg$c.json')); r=d['roofline']; print('cfg$c', round(d['value'],1), 'ms/step', round(d['ms_per_step'],5), 'stage_us', round(1000*r['avg_launch_ms'],2), 'frac', round(r['frac'],3), 'e2e', round(d['e2e']['value'],1), 'launches', d['gpu_launches'])"
done
python bench.py --impl reference --steps 2 --warmup 3 > $O/bench_reference.json 2> $O/bench_reference.err; echo reference=$?
for c in 3 5; do
  CMD="python bench.py --config $c --steps 3 --warmup 3 --no-cpu --no-e2e"
  ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches_cfg$c.csv $CMD > $O/ncu_l$c.log 2>&1; echo launches$c=$?
  python tools/launch_summary.py $O/launches_cfg$c.csv > $O/launches_cfg${c}_summary.txt 2>&1
  for k in k_stage k_remote; do
    ncu --set full --clock-control none --import-source on -k regex:$k -s 6 -c 1 -o $O/cfg${c}_$k $CMD > $O/ncu_f$c$k.log 2>&1; echo full$c$k=$?
    python tools/ncu_summary.py $O/cfg${c}_$k.ncu-rep > $O/cfg${c}_${k}_ncu_full.txt 2>&1
    python tools/ncu_stalls.py $O/cfg${c}_$k.ncu-rep 25 > $O/cfg${c}_${k}_stalls.txt 2>&1
  done
done
rm -f $O/*.ncu-rep
