# NOTE: compute-sanitizer is closed on the current GPU pool (runs under it left GPUs needing a
# reset); use the bounds-checked build instead: make debug; KUR_LIB=paper_2102_07167_b200/libkur_debug.so pytest -m gpu
mkdir -p gpurun_out
for tool in memcheck racecheck synccheck initcheck; do
  timeout 1500 compute-sanitizer --tool $tool --print-limit 20 python tools/sanitize_run.py > gpurun_out/san_$tool.log 2>&1
  echo $tool=$?; grep -E "ERROR SUMMARY|RACECHECK SUMMARY|done" gpurun_out/san_$tool.log | head -3
done
