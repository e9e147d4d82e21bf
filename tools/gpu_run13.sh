# pass 13: per-kernel A/B of the warp engine (ACRGPU_PROFILE=1)
set -x
L=$PWD/paper_1701_00182_b200
for v in old newbase old newbase; do
ACRGPU_PROFILE=1 ACRGPU_LIB=$L/libacrgpu_$v.so timeout 300 python tools/profile_run.py 2 > gpurun_out/ab3_${v}_c2_$RANDOM.log 2>&1
done
