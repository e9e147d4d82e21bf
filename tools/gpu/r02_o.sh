# A/B: CTA rrqr with 4 vs 2 columns per warp iteration (interleaved runs against box noise)
mkdir -p gpurun_out
for r in 1 2; do
  timeout 300 python tools/factor_time.py 2 - 2 | sed 's/^/{"lib": "rq4", "r": /; s/$/}/' >> gpurun_out/ab_rq.jsonl
  ACRGPU_LIB=$PWD/paper_1701_00182_b200/libacrgpu_rq2.so timeout 300 python tools/factor_time.py 2 - 2 | sed 's/^/{"lib": "rq2", "r": /; s/$/}/' >> gpurun_out/ab_rq.jsonl
done
timeout 600 python tools/factor_time.py 5 - 1 | sed 's/^/{"lib": "rq4", "r": /; s/$/}/' >> gpurun_out/ab_rq.jsonl
ACRGPU_LIB=$PWD/paper_1701_00182_b200/libacrgpu_rq2.so timeout 600 python tools/factor_time.py 5 - 1 | sed 's/^/{"lib": "rq2", "r": /; s/$/}/' >> gpurun_out/ab_rq.jsonl
timeout 2400 python tools/parity_table.py > gpurun_out/parity_table.json 2> gpurun_out/parity_table.err
