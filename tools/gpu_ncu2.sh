# ncu evidence for cfg5: launch list, --set full of k_stage and of k_remote
mkdir -p gpurun_out
CMD="python bench.py --config 5 --steps 2 --warmup 3 --no-cpu --no-e2e"
$CMD > gpurun_out/plain5.log 2>&1; echo plain=$?
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches5.csv $CMD > gpurun_out/ncu_l5.log 2>&1; echo launches=$?
ncu --set full --clock-control none --import-source on -k regex:k_stage -s 6 -c 1 -o gpurun_out/prof5 $CMD > gpurun_out/ncu_f5.log 2>&1; echo full_stage=$?
ncu --set full --clock-control none --import-source on -k regex:k_remote -s 6 -c 1 -o gpurun_out/prof5r $CMD > gpurun_out/ncu_r5.log 2>&1; echo full_remote=$?
