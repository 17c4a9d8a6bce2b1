# full evidence cycle for the current build: all GPU tests, smoke, default bench + reference line,
# cfg5 launch list, ncu --set full of k_stage and k_remote, per-tile phase profile, other configs
mkdir -p gpurun_out
timeout 2400 python -m pytest tests -q -m gpu > gpurun_out/pytest_gpu.log 2>&1; echo pytest=$?; tail -2 gpurun_out/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo smoke=$?
python bench.py > gpurun_out/bench_default.json 2> gpurun_out/bench_default.err; echo bench=$?
python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err; echo ref=$?
for c in 1 2 3 4; do python bench.py --config $c --steps 50 --warmup 3 --no-cpu > gpurun_out/b$c.json 2> gpurun_out/b$c.err; echo b$c=$?; done
python tools/tile_profile.py --config 5 > gpurun_out/tp5.log 2>&1
CMD="python bench.py --config 5 --steps 2 --warmup 3 --no-cpu --no-e2e"
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches5.csv $CMD > /dev/null 2>&1; echo launches=$?
ncu --set full --clock-control none --import-source on -k regex:k_stage -s 6 -c 1 -o gpurun_out/prof5 $CMD > /dev/null 2>&1; echo full_stage=$?
ncu --set full --clock-control none --import-source on -k regex:k_remote -s 6 -c 1 -o gpurun_out/prof5r $CMD > /dev/null 2>&1; echo full_remote=$?
