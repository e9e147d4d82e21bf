#!/bin/bash
# Round check on the GPU box: GPU suite, smoke, default bench (C2), solve roofline, per-level times,
# then the north-star system (C5) bench line, its solve, and an ncu capture of the bulk-copy slab kernel.
mkdir -p gpurun_out
python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc $?"
python __graft_entry__.py smoke > gpurun_out/smoke.log 2>&1; echo "smoke rc $?"
python bench.py > gpurun_out/bench_c2.json 2> gpurun_out/bench_c2.err; echo "bench rc $?"
python tools/solve_bench.py 2 > gpurun_out/solve_c2.json 2> gpurun_out/solve_c2.err
python tools/level_times.py 2 0 3 > gpurun_out/levels_c2.json 2>&1
if [ "$1" = "c5" ]; then
  python bench.py --config 5 --steps 2 --warmup 3 > gpurun_out/bench_c5.json 2> gpurun_out/bench_c5.err; echo "bench c5 rc $?"
  python tools/solve_bench.py 5 - 5 > gpurun_out/solve_c5.json 2> gpurun_out/solve_c5.err
  ACRGPU_MV_LDG=1 python tools/solve_bench.py 5 - 5 > gpurun_out/solve_c5_ldg.json 2> gpurun_out/solve_c5_ldg.err
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_mv_slab_tma -s 2 -c 1 -o gpurun_out/ncu_mv_slab_tma -f python tools/solve_bench.py 5 64 1 > gpurun_out/ncu_mv.log 2>&1
  timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/ncu_solve_launches_c5n64.csv -k regex:k_mv python tools/solve_bench.py 5 64 1 > gpurun_out/ncu_mv2.log 2>&1
fi
tail -3 gpurun_out/pytest_gpu.log; tail -1 gpurun_out/smoke.log; cat gpurun_out/bench_c2.json; cat gpurun_out/solve_c2.json; cat gpurun_out/levels_c2.json
