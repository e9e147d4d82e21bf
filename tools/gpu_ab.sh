#!/bin/bash
mkdir -p gpurun_out
python -m pytest tests/test_gpu_parity.py tests/test_gpu_partition.py -m gpu -x -q > gpurun_out/pytest_ab.log 2>&1; echo "pytest rc $?"; tail -5 gpurun_out/pytest_ab.log
python tools/level_times.py 2 0 4 > gpurun_out/lt_fused_c2.json 2>&1; cat gpurun_out/lt_fused_c2.json
ACRGPU_NO_FUSED_INV=1 python tools/level_times.py 2 0 3 > gpurun_out/lt_nofused_c2.json 2>&1; cat gpurun_out/lt_nofused_c2.json
python tools/level_times.py 1 0 4 > gpurun_out/lt_fused_c1.json 2>&1; cat gpurun_out/lt_fused_c1.json
python tools/profile_run.py 2 > gpurun_out/c2_fused.log 2>&1; head -1 gpurun_out/c2_fused.log | cut -c1-300
