# tile / hot_min sweep: bash tools/gpu_sweep.sh <config> "<tiles>" "<hotmins>"
C=$1
for t in $2; do for hm in $3; do
  python bench.py --config $C --steps 10 --warmup 3 --no-cpu --no-e2e --tile-rows $t --hot-min $hm > gpurun_out/sw.json 2>gpurun_out/sw.err || { echo "fail $t $hm"; tail -2 gpurun_out/sw.err; continue; }
  python -c "
import json; d=json.load(open('gpurun_out/sw.json')); r=d['roofline']; p=d['plan']
print('cfg$C tile $t hot $hm', round(d['value'],1), 'RHS/s stage_us', round(1000*r['avg_launch_ms'],2), 'tiles', p['n_tiles'], 'hot', p['n_idx_hot'], 'rem', p['n_idx_remote'])"
done; done
