# matvec v3 + host transport multiprocess test
mkdir -p gpurun_out
timeout 600 python tools/solve_bench.py 2 - 5 > gpurun_out/solve_c2_c.json 2>&1
timeout 900 python tools/solve_bench.py 5 - 3 > gpurun_out/solve_c5_c.json 2>&1
timeout 900 python -m pytest tests/test_gpu_multiprocess.py tests/test_gpu_parity.py tests/test_gpu_partition.py -m gpu -x -q > gpurun_out/pytest_c.log 2>&1; echo rc=$? >> gpurun_out/pytest_c.log
