# usage: bash tools/gpu_ncu.sh <config> <tag>   (one ncu tool per gpurun call)
C=${1:-5}; TAG=${2:-prof}
mkdir -p gpurun_out
CMD="python bench.py --config $C --steps 2 --warmup 3 --no-cpu --no-e2e"
$CMD > gpurun_out/plain_$TAG.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_$TAG.csv $CMD > gpurun_out/ncu_l_$TAG.log 2>&1; echo launches=$?
ncu --set full --clock-control none --import-source on -k regex:k_stage -s 6 -c 1 -o gpurun_out/$TAG $CMD > gpurun_out/ncu_f_$TAG.log 2>&1; echo full=$?
