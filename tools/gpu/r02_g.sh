# C5 per-kernel table (profiled warm-up step) with the current build; full GPU suite
mkdir -p gpurun_out
timeout 1200 python bench.py --config 5 --steps 1 --warmup 1 --no-e2e --no-cpu-baseline > gpurun_out/bench_c5_g.json 2> gpurun_out/bench_c5_g.err
timeout 2000 python -m pytest tests -m gpu -q > gpurun_out/pytest_g.log 2>&1; echo rc=$? >> gpurun_out/pytest_g.log
