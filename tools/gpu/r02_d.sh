# multiprocess host transport; QR-route variant A/B at C2 and C5; ncu of the solve kernels at C5
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_multiprocess.py -m gpu -x -q > gpurun_out/pytest_d.log 2>&1; echo rc=$? >> gpurun_out/pytest_d.log
for v in 0 1; do ACRGPU_QR_VARIANT=$v timeout 300 python tools/factor_time.py 2 - 3 >> gpurun_out/ab_c2.jsonl 2>&1; done
for v in 0 1; do ACRGPU_QR_VARIANT=$v timeout 600 python tools/factor_time.py 5 - 1 >> gpurun_out/ab_c5.jsonl 2>&1; done
timeout 900 ncu --kernel-name regex:k_mv --launch-count 4 --set full --clock-control none --import-source on -o gpurun_out/ncu_mv_c5 -f python tools/solve_bench.py 5 - 1 > gpurun_out/ncu_mv_c5.log 2>&1
