# pass 26: warp engine: incremental circle partner, reflector formed once in registers; C2 levels, C1
set -x
ACRGPU_VERBOSE=1 ACRGPU_PROFILE=1 timeout 300 python tools/profile_run.py 2 > gpurun_out/prof26_c2_levels.log 2>&1
ACRGPU_VERBOSE=1 timeout 300 python tools/profile_run.py 2 > gpurun_out/prof26_c2_levels_np.log 2>&1
timeout 300 python tools/profile_run.py 1 > gpurun_out/prof26_c1_np.log 2>&1
