#!/bin/bash
# Round check on the GPU box: GPU suite, smoke, default bench (C2), reference arm, solve roofline,
# per-level times, then the north-star system (C5) bench line and its solve.
mkdir -p gpurun_out
python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc $?"
python __graft_entry__.py smoke > gpurun_out/smoke.log 2>&1; echo "smoke rc $?"
python bench.py > gpurun_out/bench_c2.json 2> gpurun_out/bench_c2.err; echo "bench rc $?"
python tools/solve_bench.py 2 > gpurun_out/solve_c2.json 2>&1
python tools/level_times.py 2 0 3 > gpurun_out/levels_c2.json 2>&1
python tools/timeline.py 2 3 > gpurun_out/timeline_c2.log 2>&1
if [ "$1" = "c5" ]; then
  python bench.py --config 5 --steps 2 --warmup 3 > gpurun_out/bench_c5.json 2> gpurun_out/bench_c5.err; echo "bench c5 rc $?"
  python tools/solve_bench.py 5 - 3 > gpurun_out/solve_c5.json 2>&1
fi
tail -3 gpurun_out/pytest_gpu.log; tail -1 gpurun_out/smoke.log; cat gpurun_out/bench_c2.json; cat gpurun_out/solve_c2.json; cat gpurun_out/levels_c2.json
