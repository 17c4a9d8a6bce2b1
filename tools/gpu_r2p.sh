# bounds-checked build (in-kernel asserts on every layout index) through the parity, edge, sharded,
# persistent and methods suites
mkdir -p gpurun_out/r2p
KUR_LIB=paper_2102_07167_b200/libkur_debug.so timeout 2400 python -m pytest tests/test_gpu_parity.py tests/test_gpu_edge.py tests/test_gpu_sharded.py tests/test_gpu_persist.py tests/test_gpu_methods.py tests/test_gpu_next.py -q -m gpu > gpurun_out/r2p/pytest_gpu_debug_bounds.log 2>&1; echo dbg=$?; tail -2 gpurun_out/r2p/pytest_gpu_debug_bounds.log
