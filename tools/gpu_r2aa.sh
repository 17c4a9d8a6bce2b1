# balanced one-wave tiles for config 3 (288 tiles of 227-228 rows) vs the old 256-row tiles (--tile-rows 256)
mkdir -p gpurun_out/r2aa
O=gpurun_out/r2aa
for r in 1 2; do for tr in 0 256; do
  python bench.py --config 3 --steps 100 --warmup 5 --no-cpu --no-e2e --tile-rows $tr > $O/x.json 2> $O/x.err || { echo fail; tail -3 $O/x.err; continue; }
  python -c "import json; d=json.load(open('$O/x.json')); r=d['roofline']; print('round $r tile_rows $tr cfg3', round(d['value'],1), 'ms/step', round(d['ms_per_step'],5), 'stage_us', round(1000*r['avg_launch_ms'],2), 'tiles', d['plan']['n_tiles'])"
done; done
timeout 1500 python -m pytest tests/test_gpu_parity.py tests/test_gpu_sharded.py tests/test_gpu_methods.py tests/test_gpu_next.py -q -m gpu -x > $O/pytest.log 2>&1; echo pytest=$?; tail -3 $O/pytest.log
