# closing evidence for the round-2 HEAD build: bench lines for configs 1-4 + the reference arm, the launch
# lists of configs 5 and 3, and ncu --set full captures of k_stage / k_remote on both (each ncu pass runs
# only after the same command has exited 0 without ncu)
O=gpurun_out/fin_g
mkdir -p $O
for c in 1 2 3 4; do
  python bench.py --config $c --steps 50 --warmup 5 > $O/bench_cfg$c.json 2> $O/bench_cfg$c.err; echo cfg$c=$?
done
python bench.py --impl reference --steps 2 --warmup 3 > $O/bench_reference.json 2> $O/bench_reference.err; echo reference=$?
for c in 5 3; do
  CMD="python bench.py --config $c --steps 2 --warmup 3 --no-cpu --no-e2e"
  $CMD > $O/plain_cfg$c.json 2> $O/plain_cfg$c.err; rc=$?; echo plain$c=$rc
  [ $rc -eq 0 ] || continue
  ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches_cfg$c.csv $CMD > $O/ncu_l$c.log 2>&1; echo launches$c=$?
  ncu --set full --clock-control none --import-source on -k regex:k_stage -s 6 -c 1 -o $O/cfg${c}_k_stage $CMD > $O/ncu_s$c.log 2>&1; echo full_stage$c=$?
  ncu --set full --clock-control none --import-source on -k regex:k_remote -s 6 -c 1 -o $O/cfg${c}_k_remote $CMD > $O/ncu_r$c.log 2>&1; echo full_remote$c=$?
done
ls -la $O
# the four reports together exceed gpurun's 64 MiB return limit: summarise them on the box, keep the text
for c in 5 3; do for k in k_stage k_remote; do
  python tools/ncu_summary.py $O/cfg${c}_$k.ncu-rep > $O/cfg${c}_${k}_ncu_full.txt 2>&1
  python tools/ncu_stalls.py $O/cfg${c}_$k.ncu-rep > $O/cfg${c}_${k}_stalls.txt 2>&1
  rm -f $O/cfg${c}_$k.ncu-rep
done; python tools/launch_summary.py $O/launches_cfg$c.csv > $O/launches_cfg${c}_summary.txt 2>&1; done
du -sh $O
