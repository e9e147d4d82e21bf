# pass 33: k_deposit parts-outer / element-group-inner (records read once per part); GPU suite, C2 levels, C1
set -x
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu33.log 2>&1; echo "pytest exit $?"
ACRGPU_VERBOSE=1 timeout 300 python tools/profile_run.py 2 > gpurun_out/prof33_c2_levels_np.log 2>&1
ACRGPU_VERBOSE=1 ACRGPU_PROFILE=1 timeout 300 python tools/profile_run.py 2 > gpurun_out/prof33_c2_levels.log 2>&1
timeout 300 python tools/profile_run.py 1 > gpurun_out/prof33_c1_np.log 2>&1
