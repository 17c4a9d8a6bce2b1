# which round-2 change costs k_stage ~2 %: a = r2d build, c = current, c1 no griddepcontrol, c2 fixed window
# policy, c3 both; then the per-tile timeline of cfg3/cfg5 (prof build)
mkdir -p gpurun_out/r2j
O=gpurun_out/r2j
for r in 1 2; do for v in a c c1 c2 c3; do
  L=paper_2102_07167_b200/libkur.so; [ $v != c ] && L=paper_2102_07167_b200/libkur_$v.so
  KUR_LIB=$L python bench.py --config 5 --steps 20 --warmup 5 --no-cpu --no-e2e > $O/x.json 2> $O/x.err || { echo fail; tail -3 $O/x.err; }
  python -c "import json; d=json.load(open('$O/x.json')); r=d['roofline']; print('round $r cfg5 lib=$v', round(d['value'],1), 'ms/step', round(d['ms_per_step'],4), 'stage_us', round(1000*r['avg_launch_ms'],2), 'k_stage', round(1000*r['k_stage_ms'],2))"
done; done
python tools/tile_profile.py --config 3 > $O/tile_profile_cfg3.txt 2>&1; tail -10 $O/tile_profile_cfg3.txt
python tools/tile_profile.py --config 5 > $O/tile_profile_cfg5.txt 2>&1; tail -10 $O/tile_profile_cfg5.txt
