# cluster-resident stage: CZ tests, world-invariance suites, cfg3 A/B (KUR_CZ=0/1), occupancy
mkdir -p gpurun_out/r2z
O=gpurun_out/r2z
python -c "
import torch, sys; sys.path.insert(0,'.')
from paper_2102_07167_b200 import kur
import kurgen
g = kur.graph_build(kurgen.config(3)); print('cfg3 info', {k: g.info[k] for k in ('cluster_plan','n_tiles','rows_per_tile','n_idx_hot','n_idx_remote','n_slots_hot','n_window_loads')})
" 2>&1 | tail -3
timeout 600 python -m pytest tests/test_gpu_cluster.py -x -q -m gpu > $O/pytest_cz.log 2>&1; echo pytest_cz=$?; tail -15 $O/pytest_cz.log
for r in 1 2; do for cz in 0 1; do
  KUR_CZ=$cz python bench.py --config 3 --steps 100 --warmup 5 --no-cpu --no-e2e > $O/x.json 2> $O/x.err || { echo fail; tail -3 $O/x.err; continue; }
  python -c "import json; d=json.load(open('$O/x.json')); r=d['roofline']; print('round $r cz $cz cfg3', round(d['value'],1), 'ms/step', round(d['ms_per_step'],5), 'stage_us', round(1000*r['avg_launch_ms'],2), 'tiles', d['plan']['n_tiles'])"
done; done
timeout 1500 python -m pytest tests/test_gpu_parity.py tests/test_gpu_edge.py tests/test_gpu_methods.py tests/test_gpu_next.py tests/test_gpu_host_buffers.py tests/test_gpu_sharded.py tests/test_gpu_adaptive.py tests/test_gpu_persist.py -q -m gpu > $O/pytest.log 2>&1; echo pytest=$?; tail -15 $O/pytest.log
