# pass 12: A/B of the warp engine at 168 registers (6 CTAs/SM) vs 220 (4 CTAs/SM)
set -x
L=$PWD/paper_1701_00182_b200
for i in 1 2; do
ACRGPU_LIB=$L/libacrgpu_old.so timeout 300 python tools/profile_run.py 1 > gpurun_out/ab2_old_c1_$i.log 2>&1
ACRGPU_LIB=$L/libacrgpu_newbase.so timeout 300 python tools/profile_run.py 1 > gpurun_out/ab2_new_c1_$i.log 2>&1
done
ACRGPU_LIB=$L/libacrgpu_old.so timeout 300 python tools/profile_run.py 2 > gpurun_out/ab2_old_c2.log 2>&1
ACRGPU_LIB=$L/libacrgpu_newbase.so timeout 300 python tools/profile_run.py 2 > gpurun_out/ab2_new_c2.log 2>&1
ACRGPU_LIB=$L/libacrgpu_old.so timeout 300 python tools/profile_run.py 2 > gpurun_out/ab2_old_c2b.log 2>&1
ACRGPU_LIB=$L/libacrgpu_newbase.so timeout 300 python tools/profile_run.py 2 > gpurun_out/ab2_new_c2b.log 2>&1
