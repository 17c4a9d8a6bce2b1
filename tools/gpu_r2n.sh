# cold-window pass: tests, cfg3 A/B (KUR_NO_COLD), cfg4/cfg5 unchanged check
mkdir -p gpurun_out/r2n
O=gpurun_out/r2n
timeout 1500 python -m pytest tests/test_gpu_sharded.py tests/test_gpu_parity.py -k "cold or config3 or small or layout or remote_modes or concurrent or world_independent" -x -q -m gpu > $O/pytest.log 2>&1; echo pytest=$?; tail -3 $O/pytest.log
for r in 1 2; do for v in cold nocold; do
  [ $v = nocold ] && export KUR_NO_COLD=1
  python bench.py --config 3 --steps 50 --warmup 5 --no-cpu --no-e2e > $O/x.json 2> $O/x.err || { echo fail; tail -3 $O/x.err; }
  unset KUR_NO_COLD
  python -c "import json; d=json.load(open('$O/x.json')); r=d['roofline']; print('round $r cfg3 $v', round(d['value'],1), 'ms/step', round(d['ms_per_step'],4), 'stage_us', round(1000*r['avg_launch_ms'],2), 'k_stage', round(1000*r['k_stage_ms'],2), 'side', round(1000*r['k_remote_ms'],2))"
done; done
for c in 4 5; do
  python bench.py --config $c --steps 20 --warmup 5 --no-cpu --no-e2e > $O/x.json 2> $O/x.err || { echo fail; tail -3 $O/x.err; }
  python -c "import json; d=json.load(open('$O/x.json')); r=d['roofline']; print('cfg$c', round(d['value'],1), 'ms/step', round(d['ms_per_step'],4), 'stage_us', round(1000*r['avg_launch_ms'],2), 'cold', d['plan'].get('n_idx_cold'))"
done
