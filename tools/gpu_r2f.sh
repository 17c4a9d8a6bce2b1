mkdir -p gpurun_out/r2f
O=gpurun_out/r2f
python tools/tile_profile.py --config 3 > $O/tile_profile_cfg3.txt 2>&1; echo tp3=$?; cat $O/tile_profile_cfg3.txt | tail -8
python tools/tile_profile.py --config 5 > $O/tile_profile_cfg5.txt 2>&1; echo tp5=$?; cat $O/tile_profile_cfg5.txt | tail -8
for c in 3 4; do for rp in auto on; do
  python bench.py --config $c --steps 50 --warmup 5 --no-cpu --no-e2e --remote-pass $rp > $O/x.json 2> $O/x.err || { echo fail; tail -2 $O/x.err; continue; }
  python -c "import json; d=json.load(open('$O/x.json')); r=d['roofline']; print('cfg$c remote_pass=$rp', round(d['value'],1), 'stage_us', round(1000*r['avg_launch_ms'],2), 'k_stage', round(1000*r['k_stage_ms'],2), 'k_remote', round(1000*r['k_remote_ms'],2))"
done; done
