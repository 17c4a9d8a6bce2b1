# config 3/4 with the remote pass overlapped by k_stage (KUR_REMOTE_OVERLAP, PDL) vs inline concurrent
mkdir -p gpurun_out/r2ag
O=gpurun_out/r2ag
for r in 1 2; do for v in inline pass_ov1 pass_ov2 pass_ov3; do for c in 3 4; do
  st=20; [ $c = 3 ] && st=100
  case $v in inline) E="KUR_X=0"; RP=auto;; pass_ov1) E="KUR_REMOTE_OVERLAP=1"; RP=on;; pass_ov2) E="KUR_REMOTE_OVERLAP=2"; RP=on;; pass_ov3) E="KUR_REMOTE_OVERLAP=3"; RP=on;; esac
  env $E python bench.py --config $c --steps $st --warmup 5 --no-cpu --no-e2e --remote-pass $RP > $O/x.json 2> $O/x.err || { echo fail; tail -3 $O/x.err; continue; }
  python -c "import json; d=json.load(open('$O/x.json')); r=d['roofline']; print('round $r $v cfg$c', round(d['value'],1), 'stage_us', round(1000*r['avg_launch_ms'],2))"
done; done; done
