#!/bin/bash
mkdir -p gpurun_out
python -m pytest tests/test_gpu_parity.py tests/test_gpu_partition.py tests/test_gpu_krylov.py -m gpu -x -q > gpurun_out/pytest_ab.log 2>&1; echo "pytest rc $?"; tail -5 gpurun_out/pytest_ab.log
python tools/solve_bench.py 2 - 5 > gpurun_out/solve_c2.json 2>&1; tail -1 gpurun_out/solve_c2.json
python tools/solve_bench.py 1 - 5 > gpurun_out/solve_c1.json 2>&1; tail -1 gpurun_out/solve_c1.json
