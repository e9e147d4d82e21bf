# warp-engine DMMA formation: parity + fullsize + partition suites, C2 timing and phases
mkdir -p gpurun_out
timeout 1500 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fullsize.py tests/test_gpu_partition.py tests/test_gpu_report.py -m gpu -x -q > gpurun_out/pytest_k.log 2>&1; echo rc=$? >> gpurun_out/pytest_k.log
timeout 300 python tools/factor_time.py 2 - 2 > gpurun_out/ft_c2_k.jsonl 2>&1
timeout 300 python tools/factor_time.py 1 - 2 > gpurun_out/ft_c1_k.jsonl 2>&1
ACRGPU_PROFILE=1 timeout 300 python tools/profile_run.py 2 > gpurun_out/prof_c2_k.txt 2>&1
