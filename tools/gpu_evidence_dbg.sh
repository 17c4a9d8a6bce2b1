bash tools/gpu_evidence.sh
KUR_LIB=paper_2102_07167_b200/libkur_debug.so timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_gpu_edge.py -x -q -m gpu > gpurun_out/pt_dbg.log 2>&1; echo dbg=$?; tail -1 gpurun_out/pt_dbg.log
