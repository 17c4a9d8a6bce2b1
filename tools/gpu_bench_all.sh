set -x
python bench.py --steps 20 --warmup 3 > gpurun_out/b5.json 2> gpurun_out/b5.err; echo b5=$?
for c in 1 2 3 4; do python bench.py --config $c --steps 50 --warmup 3 --no-cpu > gpurun_out/b$c.json 2> gpurun_out/b$c.err; echo b$c=$?; done
python bench.py --steps 2 --warmup 3 --no-cpu --no-e2e > gpurun_out/plain5.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches5.csv python bench.py --steps 2 --warmup 3 --no-cpu --no-e2e > gpurun_out/ncu_l5.log 2>&1; echo ncu1=$?
ncu --set full --clock-control none --import-source on -k regex:k_stage -s 6 -c 1 -o gpurun_out/prof5 python bench.py --steps 2 --warmup 3 --no-cpu --no-e2e > gpurun_out/ncu_f5.log 2>&1; echo ncu2=$?
