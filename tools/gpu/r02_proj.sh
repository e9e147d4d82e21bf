# C5 sub-system level times for the 2/4/8-GPU projection + CTA rrqr 4-column change timing/tests
mkdir -p gpurun_out
for k in 16 32 64; do timeout 900 python tools/level_times.py 5 $k 2 > gpurun_out/proj_c5_p$k.json 2>&1; done
timeout 900 python tools/level_times.py 5 0 2 > gpurun_out/proj_c5_full.json 2>&1
timeout 300 python tools/factor_time.py 2 - 3 > gpurun_out/ft_c2_n.jsonl 2>&1
timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fullsize.py -m gpu -x -q > gpurun_out/pytest_n.log 2>&1; echo rc=$? >> gpurun_out/pytest_n.log
