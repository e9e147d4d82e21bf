# pass 18: warp-parallel condition estimate + inverse in k_lu_inverse: GPU suite, timings
set -x
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu18.log 2>&1; echo "pytest exit $?"
ACRGPU_PROFILE=1 timeout 300 python tools/profile_run.py 2 > gpurun_out/prof18_c2.log 2>&1
for i in 1 2; do timeout 300 python tools/profile_run.py 2 > gpurun_out/prof18_c2_np_$i.log 2>&1; timeout 300 python tools/profile_run.py 1 > gpurun_out/prof18_c1_np_$i.log 2>&1; done
