mkdir -p gpurun_out/r2g
O=gpurun_out/r2g
python tools/tile_profile.py --config 3 > $O/tile_profile_cfg3.txt 2>&1; cat $O/tile_profile_cfg3.txt | tail -9
python tools/tile_profile.py --config 3 --tile-rows 128 > $O/tile_profile_cfg3_128.txt 2>&1; cat $O/tile_profile_cfg3_128.txt | tail -9
for tr in 128 192; do
  python bench.py --config 3 --steps 50 --warmup 5 --no-cpu --no-e2e --tile-rows $tr > $O/x.json 2> $O/x.err || { echo fail; tail -2 $O/x.err; continue; }
  python -c "import json; d=json.load(open('$O/x.json')); r=d['roofline']; print('cfg3 tile $tr', round(d['value'],1), 'stage_us', round(1000*r['avg_launch_ms'],2), d['plan']['n_tiles'])"
done
