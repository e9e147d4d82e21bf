#!/bin/bash
mkdir -p gpurun_out
python tools/timeline.py 2 3 > gpurun_out/c2_tl.log 2>&1
grep "timeline\|factor_ms" gpurun_out/c2_tl.log
