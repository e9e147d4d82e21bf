# DMMA warp-per-item apply kernels: full GPU suite (verbose), C2/C5 timing + phase breakdown
mkdir -p gpurun_out
timeout 2000 python -m pytest tests -m gpu -q -rs > gpurun_out/pytest_i.log 2>&1; echo rc=$? >> gpurun_out/pytest_i.log
timeout 300 python tools/factor_time.py 2 - 2 > gpurun_out/ft_c2_i.jsonl 2>&1
ACRGPU_PROFILE=1 timeout 300 python tools/profile_run.py 2 > gpurun_out/prof_c2_i.txt 2>&1
timeout 600 python tools/factor_time.py 5 - 1 > gpurun_out/ft_c5_i.jsonl 2>&1
