# pass 8: two-CTA mid64 truncation; full GPU suite incl. the C5-operator (leaf 64, 16 RHS) parity test
set -x
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu8.log 2>&1; echo "pytest exit $?"
timeout 300 python tools/profile_run.py 2 > gpurun_out/prof_c2_r8.log 2>&1; echo "c2 exit $?"
timeout 300 python tools/profile_run.py 1 > gpurun_out/prof_c1_r8.log 2>&1; echo "c1 exit $?"
