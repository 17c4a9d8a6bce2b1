# tile / hot_min / remote-pass sweep: bash tools/gpu_sweep2.sh <config> "<tiles>" "<hotmins>" "<remote: auto on off>"
C=$1
for t in $2; do for hm in $3; do for rp in ${4:-auto}; do
  python bench.py --config $C --steps 20 --warmup 3 --no-cpu --no-e2e --tile-rows $t --hot-min $hm --remote-pass $rp > gpurun_out/sw.json 2>gpurun_out/sw.err || { echo "fail $t $hm $rp"; tail -2 gpurun_out/sw.err; continue; }
  python -c "
import json; d=json.load(open('gpurun_out/sw.json')); r=d['roofline']; p=d['plan']
print('cfg$C tile $t hot $hm rp $rp', round(d['value'],1), 'RHS/s stage_us', round(1000*r['avg_launch_ms'],2), 'tiles', p['n_tiles'], 'hot', p['n_idx_hot'], 'rem', p['n_idx_remote'])"
done; done; done
