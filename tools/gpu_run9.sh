# pass 9: A/B of the warp-engine register cap (k_small32 __launch_bounds__(64, 5)) at C1 and C2
set -x
for i in 1 2; do
timeout 300 python tools/profile_run.py 1 > gpurun_out/ab_base_c1_$i.log 2>&1
ACRGPU_LIB=$PWD/paper_1701_00182_b200/libacrgpu_k5.so timeout 300 python tools/profile_run.py 1 > gpurun_out/ab_k5_c1_$i.log 2>&1
done
timeout 300 python tools/profile_run.py 2 > gpurun_out/ab_base_c2.log 2>&1
ACRGPU_LIB=$PWD/paper_1701_00182_b200/libacrgpu_k5.so timeout 300 python tools/profile_run.py 2 > gpurun_out/ab_k5_c2.log 2>&1
