mkdir -p gpurun_out/r2k
O=gpurun_out/r2k
timeout 2000 python -m pytest tests/test_gpu_parity.py tests/test_gpu_edge.py tests/test_gpu_sharded.py tests/test_gpu_persist.py tests/test_gpu_next.py -x -q -m gpu > $O/pytest.log 2>&1; echo pytest=$?; tail -2 $O/pytest.log
for r in 1 2; do for c in 3 4 5; do for v in a c lpt; do
  L=paper_2102_07167_b200/libkur.so; [ $v = a ] && L=paper_2102_07167_b200/libkur_a.so
  [ $v = lpt ] && export KUR_TILE_ORDER=lpt
  KUR_LIB=$L python bench.py --config $c --steps 20 --warmup 5 --no-cpu --no-e2e > $O/x.json 2> $O/x.err || { echo fail; tail -3 $O/x.err; }
  unset KUR_TILE_ORDER
  python -c "import json; d=json.load(open('$O/x.json')); r=d['roofline']; print('round $r cfg$c lib=$v', round(d['value'],1), 'ms/step', round(d['ms_per_step'],4), 'stage_us', round(1000*r['avg_launch_ms'],2), 'k_stage', round(1000*r['k_stage_ms'],2))"
done; done; done
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sector_hit_rate.pct --cache-control none --clock-control none -k regex:k_stage -s 10 -c 2 --csv python bench.py --config 5 --steps 2 --warmup 3 --no-cpu --no-e2e > $O/ncu_warm_cfg5.csv 2> $O/ncu_warm_cfg5.err
grep -E "dram__bytes_read|gpu__time|hit_rate" $O/ncu_warm_cfg5.csv | awk -F'","' '{print "   ", $(NF-3), $(NF-2), $NF}' | tail -6
python tools/tile_profile.py --config 3 > $O/tile_profile_cfg3.txt 2>&1; tail -10 $O/tile_profile_cfg3.txt
