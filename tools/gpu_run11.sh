# pass 11: GPU Krylov drivers (pcg / iterative refinement) vs the oracle
set -x
timeout 900 python -m pytest tests/test_gpu_krylov.py -m gpu -x -q > gpurun_out/pytest_krylov.log 2>&1; echo "pytest exit $?"
