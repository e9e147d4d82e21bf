# DMMA dd formation + DMMA deposit: parity subset, C2/C5 timing, CTA-engine phase breakdown
mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fullsize.py tests/test_gpu_partition.py -m gpu -x -q > gpurun_out/pytest_h.log 2>&1; echo rc=$? >> gpurun_out/pytest_h.log
timeout 300 python tools/factor_time.py 2 - 2 > gpurun_out/ft_c2_h.jsonl 2>&1
ACRGPU_PROFILE=1 timeout 300 python tools/profile_run.py 2 > gpurun_out/prof_c2_h.txt 2>&1
timeout 600 python tools/factor_time.py 5 - 1 > gpurun_out/ft_c5_h.jsonl 2>&1
ACRGPU_PROFILE=1 timeout 600 python tools/profile_run.py 5 > gpurun_out/prof_c5_h.txt 2>&1
