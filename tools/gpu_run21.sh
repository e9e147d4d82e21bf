# pass 21: per-level kernel breakdown at C2, levels without profiling, ncu launch list of the C2 bench command
set -x
ACRGPU_VERBOSE=1 ACRGPU_PROFILE=1 timeout 300 python tools/profile_run.py 2 > gpurun_out/prof21_c2_levels.log 2>&1
ACRGPU_VERBOSE=1 timeout 300 python tools/profile_run.py 2 > gpurun_out/prof21_c2_levels_np.log 2>&1
timeout 300 python tools/profile_run.py 2 > gpurun_out/prof21_c2_np.log 2>&1
timeout 1200 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file /tmp/launches_c2.csv python bench.py --steps 1 --warmup 0 --no-e2e --no-cpu-baseline > gpurun_out/ncu21.log 2>&1; echo "ncu $?"
gzip -c /tmp/launches_c2.csv > gpurun_out/r21_ncu_launches_c2.csv.gz
python tools/launch_shares.py /tmp/launches_c2.csv > gpurun_out/r21_launch_shares_c2.txt 2>&1
