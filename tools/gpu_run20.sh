# pass 20: report/CLI/ledger GPU tests + reference generators vs oracle
set -x
timeout 900 python -m pytest tests/test_gpu_report.py -x -q > gpurun_out/pytest_gpu20_report.log 2>&1; echo "pytest report exit $?"
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu20.log 2>&1; echo "pytest all exit $?"
