# plan cache across factorizations: host enqueue vs device time, C2/C1 (4 reps), C5 (2 reps)
mkdir -p gpurun_out
ACRGPU_VERBOSE=1 timeout 300 python tools/factor_time.py 2 - 4 > gpurun_out/m_c2.jsonl 2> gpurun_out/m_c2.err
ACRGPU_VERBOSE=1 timeout 300 python tools/factor_time.py 1 - 4 > gpurun_out/m_c1.jsonl 2> gpurun_out/m_c1.err
ACRGPU_VERBOSE=1 timeout 900 python tools/factor_time.py 5 - 2 > gpurun_out/m_c5.jsonl 2> gpurun_out/m_c5.err
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_partition.py tests/test_gpu_multiprocess.py -m gpu -x -q > gpurun_out/pytest_m.log 2>&1; echo rc=$? >> gpurun_out/pytest_m.log
