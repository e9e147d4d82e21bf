# pass 16: ncu --set full of the reworked small kernels at C2 level-0 sized launches
set -x
timeout 900 ncu --set full --clock-control none --import-source on --kernel-name-base demangled -k "regex:k_small32<\(int\)1>" -s 300 -c 1 -o gpurun_out/r16_dd32_c2 python tools/profile_run.py 2 > gpurun_out/ncu16a.log 2>&1; echo "a $?"
timeout 900 ncu --set full --clock-control none --import-source on --kernel-name-base demangled -k "regex:k_truncate<\(int\)64" -s 100 -c 1 -o gpurun_out/r16_mid64_c2 python tools/profile_run.py 2 > gpurun_out/ncu16b.log 2>&1; echo "b $?"
timeout 900 ncu --set full --clock-control none --import-source on --kernel-name-base demangled -k "regex:k_truncate<\(int\)128" -s 60 -c 3 -o gpurun_out/r16_big_c2 python tools/profile_run.py 2 > gpurun_out/ncu16c.log 2>&1; echo "c $?"
