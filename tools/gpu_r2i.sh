# cfg5 k_stage: L2 policy of the window loads x tile launch order; time (bench) + DRAM bytes (ncu, warm L2)
mkdir -p gpurun_out/r2i
O=gpurun_out/r2i
for r in 1 2; do for c in 3 4 5; do for v in a c; do
  L=paper_2102_07167_b200/libkur.so; [ $v = a ] && L=paper_2102_07167_b200/libkur_a.so
  KUR_LIB=$L python bench.py --config $c --steps 20 --warmup 5 --no-cpu --no-e2e > $O/x.json 2> $O/x.err || { echo fail; tail -3 $O/x.err; }
  python -c "import json; d=json.load(open('$O/x.json')); r=d['roofline']; print('round $r cfg$c lib=$v', round(d['value'],1), 'ms/step', round(d['ms_per_step'],4), 'stage_us', round(1000*r['avg_launch_ms'],2))"
done; done; done
for r in 1 2; do for v in "0 0" "1 0" "2 0" "0 1" "1 1"; do
  set -- $v
  export KUR_WIN_POLICY=$1; if [ $2 = 1 ]; then export KUR_TILE_ORDER_PLAIN=1; fi
  python bench.py --config 5 --steps 20 --warmup 5 --no-cpu --no-e2e > $O/x.json 2> $O/x.err || { echo fail; tail -3 $O/x.err; }
  python -c "import json; d=json.load(open('$O/x.json')); r=d['roofline']; print('round $r win_policy=$1 plain_order=$2', round(d['value'],1), 'stage_us', round(1000*r['avg_launch_ms'],2), 'k_stage', round(1000*r['k_stage_ms'],2))"
  if [ $r = 1 ]; then
    ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sector_hit_rate.pct --cache-control none --clock-control none -k regex:k_stage -s 10 -c 2 --csv python bench.py --config 5 --steps 2 --warmup 3 --no-cpu --no-e2e > $O/ncu_w$1_o$2.csv 2> $O/ncu_w$1_o$2.err
    grep -E "dram__bytes_read|gpu__time|hit_rate" $O/ncu_w$1_o$2.csv | awk -F'","' '{print "   ", $(NF-3), $(NF-2), $NF}' | tail -6
  fi
  unset KUR_WIN_POLICY KUR_TILE_ORDER_PLAIN
done; done
