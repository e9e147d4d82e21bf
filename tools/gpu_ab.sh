#!/bin/bash
mkdir -p gpurun_out
python tools/solve_bench.py 2 - 3 > gpurun_out/solve_plain.log 2>&1 || exit 1
tail -1 gpurun_out/solve_plain.log
ncu --set full --clock-control none --import-source on -k "regex:k_mv_t1|k_mv_slab1" -s 70 -c 8 -o gpurun_out/prof_mv1 python tools/solve_bench.py 2 - 1 > gpurun_out/ncu2.log 2>&1
ncu --set full --clock-control none --import-source on -k "regex:k_apply|k_deposit|k_lu_inverse|k_alloc_apply" -s 2500 -c 10 -o gpurun_out/prof_small python tools/profile_run.py 2 > gpurun_out/ncu3.log 2>&1
python tools/level_times.py 2 0 4 > gpurun_out/levels_c2_lu.json 2>&1; cat gpurun_out/levels_c2_lu.json
python tools/level_times.py 1 0 4 > gpurun_out/levels_c1_lu.json 2>&1; cat gpurun_out/levels_c1_lu.json
