# pass 15: copy-engine counter resets, one-CTA-per-item apply/deposit restored
set -x
for i in 1 2; do
timeout 300 python tools/profile_run.py 2 > gpurun_out/prof15_c2_noprof_$i.log 2>&1
done
ACRGPU_PROFILE=1 timeout 300 python tools/profile_run.py 2 > gpurun_out/prof15_c2.log 2>&1
timeout 600 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "config1_full or deterministic or compaction or multi_rhs" > gpurun_out/pytest15.log 2>&1; echo "pytest exit $?"
