# pass 3: C2 arena use, ncu full captures of the small-block kernels (C1), C5 memory attempt
set -x
ACRGPU_ARENA_STATS=1 timeout 300 python tools/profile_run.py 2 > gpurun_out/prof_c2_arena.log 2>&1; echo "c2 arena exit $?"
timeout 600 ncu --set full --clock-control none --import-source on --kernel-name-base demangled -k "regex:k_small32<1>" -s 20 -c 1 -o gpurun_out/k_dd_small32_c1 python tools/profile_run.py 1 > gpurun_out/ncu_dd.log 2>&1; echo "ncu dd exit $?"
timeout 600 ncu --set full --clock-control none --import-source on --kernel-name-base demangled -k "regex:k_truncate<64" -s 20 -c 1 -o gpurun_out/k_mid64_c1 python tools/profile_run.py 1 > gpurun_out/ncu_mid.log 2>&1; echo "ncu mid exit $?"
ACRGPU_PERSIST_FRAC=0.40 ACRGPU_TRANS_FRAC=0.16 ACRGPU_ARENA_STATS=1 ACRGPU_VERBOSE=1 timeout 1800 python tools/profile_run.py 5 > gpurun_out/prof_c5.log 2>&1; echo "c5 exit $?"
