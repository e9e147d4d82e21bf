# measured CPU baseline on the GPU box's host (oracle restatement of the reference path):
# C2 full size with all host threads (plane-parallel, parallel.cpp:383-405) + the bench's
# n=16 extrapolation sample (calibration), and C1 full size on one core (sequential)
mkdir -p gpurun_out
nproc > gpurun_out/cpu_nproc.txt; grep -m1 "model name" /proc/cpuinfo >> gpurun_out/cpu_nproc.txt
P=$(nproc)
timeout 3000 python tools/cpu_baseline.py 2 $P --sample-n 16 > gpurun_out/cpu_c2_p$P.json 2>&1
timeout 1500 python tools/cpu_baseline.py 1 1 > gpurun_out/cpu_c1_p1.json 2>&1
