#!/bin/bash
mkdir -p gpurun_out
ACRGPU_VERBOSE=1 python tools/profile_run.py 5 > gpurun_out/c5_mid.log 2>&1
grep "rank 0 level" gpurun_out/c5_mid.log | tr '\n' ' '; grep -o '"res": [^,]*\|"factor_ms": [^,]*\|"avg": [^,]*' gpurun_out/c5_mid.log
python -m pytest tests/test_gpu_fullsize.py tests/test_gpu_parity.py -m gpu -x -q > gpurun_out/pytest_ab.log 2>&1; echo "pytest rc $?"; tail -5 gpurun_out/pytest_ab.log
