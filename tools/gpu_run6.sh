# pass 6: C2 bench after the zero-operand skip; profiling-event overhead check; ncu captures of dd/mid64 (C1)
set -x
timeout 900 python bench.py --no-cpu-baseline > gpurun_out/bench_c2_r6.json 2> gpurun_out/bench_c2_r6.err; echo "bench exit $?"
timeout 300 python tools/profile_run.py 2 > gpurun_out/prof_c2_noprof.log 2>&1; echo "noprof exit $?"
timeout 600 ncu --set full --clock-control none --import-source on --kernel-name-base demangled -k "regex:k_small32<\(int\)1>" -s 40 -c 1 -o gpurun_out/k_dd_small32_c1 python tools/profile_run.py 1 > gpurun_out/ncu_dd.log 2>&1; echo "ncu dd exit $?"
timeout 600 ncu --set full --clock-control none --import-source on --kernel-name-base demangled -k "regex:k_truncate<\(int\)64" -s 20 -c 1 -o gpurun_out/k_mid64_c1 python tools/profile_run.py 1 > gpurun_out/ncu_mid.log 2>&1; echo "ncu mid exit $?"
