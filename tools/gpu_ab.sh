#!/bin/bash
mkdir -p gpurun_out
ACRGPU_PIPELINE_BIG=1 ACRGPU_VERBOSE=1 timeout 900 python tools/profile_run.py 5 > gpurun_out/c5_pipe.log 2>&1; echo rc $?
grep "timeline\|rank 0 level\|compaction" gpurun_out/c5_pipe.log | cut -c1-700; grep -o '"res": [^,]*\|"factor_ms": [^,]*\|"avg": [^,]*' gpurun_out/c5_pipe.log; tail -3 gpurun_out/c5_pipe.log | cut -c1-300
