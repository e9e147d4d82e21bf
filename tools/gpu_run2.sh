# round-1 measurement pass 2: per-level timing at C2, C1 bench + its ncu launch list, C5 attempt
set -x
ACRGPU_VERBOSE=1 timeout 300 python tools/profile_run.py 2 > gpurun_out/prof_c2_levels.log 2>&1; echo "lev exit $?"
timeout 300 python bench.py --config 1 > gpurun_out/bench_c1.json 2> gpurun_out/bench_c1.err; echo "bench c1 exit $?"
timeout 1500 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_c1.csv python bench.py --config 1 --steps 1 --warmup 0 --no-e2e --no-cpu-baseline > gpurun_out/ncu_launch_c1.log 2>&1; echo "ncu c1 exit $?"
nvidia-smi --query-gpu=memory.total,memory.used --format=csv
ACRGPU_VERBOSE=1 ACRGPU_ARENA_STATS=1 timeout 1500 python tools/profile_run.py 5 > gpurun_out/prof_c5.log 2>&1; echo "c5 exit $?"
