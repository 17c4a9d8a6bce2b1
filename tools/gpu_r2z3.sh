# cluster-resident stage, cross-chunk pipelined parts: CZ tests, cfg3 A/B, ncu of k_stage_cz
mkdir -p gpurun_out/r2z3
O=gpurun_out/r2z3
timeout 600 python -m pytest tests/test_gpu_cluster.py -x -q -m gpu > $O/pytest_cz.log 2>&1; echo pytest_cz=$?; tail -3 $O/pytest_cz.log
for r in 1 2; do for cz in 0 1; do
  KUR_CZ=$cz python bench.py --config 3 --steps 100 --warmup 5 --no-cpu --no-e2e > $O/x.json 2> $O/x.err || { echo fail; tail -3 $O/x.err; continue; }
  python -c "import json; d=json.load(open('$O/x.json')); r=d['roofline']; print('round $r cz $cz cfg3', round(d['value'],1), 'ms/step', round(d['ms_per_step'],5), 'stage_us', round(1000*r['avg_launch_ms'],2), 'tiles', d['plan']['n_tiles'])"
done; done
CMD="python bench.py --config 3 --steps 3 --warmup 3 --no-cpu --no-e2e"
ncu --set full --clock-control none --import-source on -k regex:k_stage_cz -s 6 -c 1 -o $O/cfg3_cz $CMD > $O/ncu_f3.log 2>&1; echo full3=$?
python tools/ncu_stalls.py $O/cfg3_cz.ncu-rep 30 > $O/cfg3_cz_stalls.txt 2>&1; head -40 $O/cfg3_cz_stalls.txt
