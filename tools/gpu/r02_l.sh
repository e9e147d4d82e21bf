# host-boundness: C2/C1 with and without the intra-mult_add fork/join, host enqueue time per factor
mkdir -p gpurun_out
nproc > gpurun_out/l_host.txt; grep -m1 "model name" /proc/cpuinfo >> gpurun_out/l_host.txt; uptime >> gpurun_out/l_host.txt
for f in 0 1; do
  if [ $f = 1 ]; then export ACRGPU_NO_FORK=1; fi
  ACRGPU_VERBOSE=1 timeout 300 python tools/factor_time.py 2 - 3 > gpurun_out/l_c2_nofork$f.jsonl 2> gpurun_out/l_c2_nofork$f.err
  ACRGPU_VERBOSE=1 timeout 300 python tools/factor_time.py 1 - 3 > gpurun_out/l_c1_nofork$f.jsonl 2> gpurun_out/l_c1_nofork$f.err
done
