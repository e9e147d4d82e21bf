set -x
timeout 600 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "compaction or deterministic" > gpurun_out/pytest_gc.log 2>&1; echo "pytest exit $?"
ACRGPU_VERBOSE=1 ACRGPU_ARENA_STATS=1 timeout 1500 python tools/profile_run.py 5 > gpurun_out/prof_c5.log 2>&1; echo "c5 exit $?"
bash tools/gpu_run6.sh
