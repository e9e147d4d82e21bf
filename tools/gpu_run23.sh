# pass 23: bqr slice-fold (QR-route kernel 73k -> 33k SASS) + warp-engine phase counters; per-level kernels at C2
set -x
ACRGPU_VERBOSE=1 ACRGPU_PROFILE=1 timeout 300 python tools/profile_run.py 2 > gpurun_out/prof23_c2_levels.log 2>&1
ACRGPU_VERBOSE=1 timeout 300 python tools/profile_run.py 2 > gpurun_out/prof23_c2_levels_np.log 2>&1
timeout 300 python tools/profile_run.py 1 > gpurun_out/prof23_c1_np.log 2>&1
