# pass 22: rolled warp engine (code size 42k -> 9k SASS): C2/C1 timing per level, bitwise check, GPU suite
set -x
ACRGPU_VERBOSE=1 timeout 300 python tools/profile_run.py 2 > gpurun_out/prof22_c2_levels_np.log 2>&1
ACRGPU_VERBOSE=1 ACRGPU_PROFILE=1 timeout 300 python tools/profile_run.py 2 > gpurun_out/prof22_c2_levels.log 2>&1
timeout 300 python tools/profile_run.py 1 > gpurun_out/prof22_c1_np.log 2>&1
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu22.log 2>&1; echo "pytest exit $?"
