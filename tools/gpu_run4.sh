# pass 4: C5 on one GPU with persistent-arena compaction; C2 regression check
set -x
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu4.log 2>&1; echo "pytest exit $?"
ACRGPU_VERBOSE=1 ACRGPU_ARENA_STATS=1 timeout 300 python tools/profile_run.py 2 > gpurun_out/prof_c2_gc.log 2>&1; echo "c2 exit $?"
ACRGPU_VERBOSE=1 ACRGPU_ARENA_STATS=1 timeout 2400 python tools/profile_run.py 5 > gpurun_out/prof_c5.log 2>&1; echo "c5 exit $?"
