# cfg3: tile size x window staging threshold (the remote entries of other communities become hot)
mkdir -p gpurun_out/sw3
for tr_hm in "0 0" "256 1024" "256 512" "512 2048" "512 1024" "1024 2048" "512 768"; do
  set -- $tr_hm
  python bench.py --config 3 --steps 50 --warmup 5 --no-cpu --no-e2e --tile-rows $1 --hot-min $2 > gpurun_out/sw3/x.json 2> gpurun_out/sw3/x.err || { echo fail $1 $2; tail -2 gpurun_out/sw3/x.err; continue; }
  python -c "import json; d=json.load(open('gpurun_out/sw3/x.json')); r=d['roofline']; print('cfg3 tile $1 hot_min $2', round(d['value'],1), 'stage_us', round(1000*r['avg_launch_ms'],2), d['plan']['n_tiles'], d['plan']['n_idx_remote'])"
done
