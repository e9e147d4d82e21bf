mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/smi.txt 2>&1
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest.log 2>&1; echo rc=$? >> gpurun_out/pytest.log
timeout 300 python tools/solve_bench.py 2 - 5 > gpurun_out/solve_c2.json 2>&1
timeout 600 python bench.py --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/bench_c2.json 2>gpurun_out/bench_c2.err
timeout 600 python tools/solve_bench.py 5 - 3 > gpurun_out/solve_c5.json 2>&1
