# pass 14: grid-stride apply/deposit kernels + 168-register warp engine: GPU suite, per-kernel C2 profile, C1/C2 timing
set -x
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu14.log 2>&1; echo "pytest exit $?"
ACRGPU_PROFILE=1 timeout 300 python tools/profile_run.py 2 > gpurun_out/prof14_c2.log 2>&1
timeout 300 python tools/profile_run.py 2 > gpurun_out/prof14_c2_noprof.log 2>&1
timeout 300 python tools/profile_run.py 1 > gpurun_out/prof14_c1_noprof.log 2>&1
