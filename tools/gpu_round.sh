#!/bin/bash
# Round check on the GPU box: GPU suite, smoke, default bench, solve roofline, per-level times.
mkdir -p gpurun_out
python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc $?"
python __graft_entry__.py smoke > gpurun_out/smoke.log 2>&1; echo "smoke rc $?"
python bench.py > gpurun_out/bench_c2.json 2> gpurun_out/bench_c2.err; echo "bench rc $?"
python tools/solve_bench.py 2 > gpurun_out/solve_c2.json 2>&1
python tools/level_times.py 2 0 2 > gpurun_out/levels_c2.json 2>&1
tail -3 gpurun_out/pytest_gpu.log; cat gpurun_out/smoke.log | tail -1; cat gpurun_out/bench_c2.json; cat gpurun_out/solve_c2.json; cat gpurun_out/levels_c2.json
