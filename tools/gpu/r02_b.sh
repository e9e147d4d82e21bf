# solve kernels v2 + async gc watermark: parity subset, solve roofline, C5 level times
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_partition.py tests/test_gpu_krylov.py -m gpu -x -q > gpurun_out/pytest_b.log 2>&1; echo rc=$? >> gpurun_out/pytest_b.log
timeout 300 python tools/solve_bench.py 2 - 5 > gpurun_out/solve_c2_b.json 2>&1
ACRGPU_VERBOSE=1 timeout 900 python tools/solve_bench.py 5 - 3 > gpurun_out/solve_c5_b.json 2> gpurun_out/c5_levels_b.log
