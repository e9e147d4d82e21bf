# pass 28b: Jacobi stop at 1e-3 eps (truncating engines): parity suite, C2 / C1 levels + warp-engine sweeps
set -x
ACRGPU_VERBOSE=1 ACRGPU_PROFILE=1 timeout 300 python tools/profile_run.py 2 > gpurun_out/prof28b_c2_levels.log 2>&1
ACRGPU_VERBOSE=1 timeout 300 python tools/profile_run.py 2 > gpurun_out/prof28b_c2_levels_np.log 2>&1
timeout 300 python tools/profile_run.py 1 > gpurun_out/prof28b_c1_np.log 2>&1
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu28b.log 2>&1; echo "pytest exit $?"
