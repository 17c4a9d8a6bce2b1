# k_stage overlapping the k_remote pass (PDL dependent, wait before the finalize): cfg5 A/B + parity
mkdir -p gpurun_out/r2ab
O=gpurun_out/r2ab
for r in 1 2; do for ov in 0 1 2; do
  KUR_REMOTE_OVERLAP=$ov python bench.py --config 5 --steps 20 --warmup 5 --no-cpu --no-e2e > $O/x.json 2> $O/x.err || { echo fail; tail -3 $O/x.err; continue; }
  python -c "import json; d=json.load(open('$O/x.json')); r=d['roofline']; print('round $r overlap $ov cfg5', round(d['value'],1), 'ms/step', round(d['ms_per_step'],5), 'stage_us', round(1000*r['avg_launch_ms'],2))"
done; done
KUR_REMOTE_OVERLAP=1 timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_gpu_sharded.py -q -m gpu -x -k "config5 or remote or bitwise" > $O/pytest.log 2>&1; echo pytest=$?; tail -3 $O/pytest.log
