# dense-route vs QR-route K threshold for blocks <= 128 (ACRGPU_DENSE_MIN_K): C2 and C5 factor times
mkdir -p gpurun_out
for t in 0 32 64 128; do ACRGPU_DENSE_MIN_K=$t timeout 300 python tools/factor_time.py 2 - 2 | sed "s/^/{\"kmin\": $t, \"r\": /; s/$/}/" >> gpurun_out/ab_kmin_c2.jsonl 2>&1; done
for t in 0 64 128; do ACRGPU_DENSE_MIN_K=$t timeout 600 python tools/factor_time.py 5 - 1 | sed "s/^/{\"kmin\": $t, \"r\": /; s/$/}/" >> gpurun_out/ab_kmin_c5.jsonl 2>&1; done
