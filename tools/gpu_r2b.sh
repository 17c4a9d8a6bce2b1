# round-2 second check: persistent entry-free kernel + gather4 remote warp (parity), cfg5 A/B of
# the remote modes, cfg1-4 bench lines with the oracle protocol, ncu evidence for cfg2-4
mkdir -p gpurun_out/r2b
O=gpurun_out/r2b
timeout 1200 python -m pytest tests/test_gpu_persist.py "tests/test_gpu_sharded.py::test_remote_modes_bitwise" tests/test_gpu_parity.py -k "persist or remote_modes or config2 or complete or spec or order_parameter" -x -q -m gpu > $O/pytest.log 2>&1; echo pytest=$?; tail -3 $O/pytest.log
for r in 1 2; do for m in b 0 3; do
  L=paper_2102_07167_b200/libkur.so; [ $m = b ] && L=paper_2102_07167_b200/libkur_b.so
  KUR_LIB=$L KUR_REMOTE_MODE=$m python bench.py --config 5 --steps 20 --warmup 3 --no-cpu --no-e2e > $O/ab.json 2> $O/ab.err || { echo fail $m; tail -3 $O/ab.err; continue; }
  python -c "
import json; d=json.load(open('$O/ab.json')); r=d['roofline']; print('round $r mode$m', round(d['value'],1), 'stage_us', round(1000*r['avg_launch_ms'],2), 'k_stage_us', round(1000*(r.get('k_stage_ms') or 0),2), 'k_remote_us', round(1000*(r.get('k_remote_ms') or 0),2), d['clocks']['sm_mhz'])"
done; done
for p in 1 0; do
  if [ $p = 0 ]; then export KUR_NO_PERSIST=1; fi
  python bench.py --config 2 --steps 200 --warmup 5 --no-cpu > $O/cfg2_p$p.json 2> $O/cfg2_p$p.err; echo cfg2 persist=$p rc=$?
  python -c "import json; d=json.load(open('$O/cfg2_p$p.json')); print('cfg2 persist=$p', round(d['value'],1), 'ms/step', round(d['ms_per_step'],5), 'e2e', round(d['e2e']['value'],1), 'rhs_calls', round(d['rhs_calls']['value'],1))"
  unset KUR_NO_PERSIST
done
for c in 1 2 3 4; do
  python bench.py --config $c --steps 50 --warmup 5 > $O/bench_cfg$c.json 2> $O/bench_cfg$c.err; echo bench cfg$c rc=$?
  python -c "import json; d=json.load(open('$O/bench_cfg$c.json')); r=d['roofline']; print('cfg$c', round(d['value'],1), 'stage_us', round(1000*r['avg_launch_ms'],2), 'frac', round(r['frac'],3), 'e2e', round(d['e2e']['value'],1), 'cpu', d['cpu_baseline']['value'])"
done
for c in 2 3 4; do
  CMD="python bench.py --config $c --steps 3 --warmup 3 --no-cpu --no-e2e"
  ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches_cfg$c.csv $CMD > $O/ncu_l$c.log 2>&1; echo launches$c=$?
done
ncu --set full --clock-control none --import-source on -k regex:k_persist -c 1 -o $O/cfg2_persist python bench.py --config 2 --steps 3 --warmup 3 --no-cpu --no-e2e > $O/ncu_f2.log 2>&1; echo full2=$?
for c in 3 4; do
  ncu --set full --clock-control none --import-source on -k regex:k_stage -s 6 -c 1 -o $O/cfg${c}_stage python bench.py --config $c --steps 2 --warmup 3 --no-cpu --no-e2e > $O/ncu_f$c.log 2>&1; echo full$c=$?
done
