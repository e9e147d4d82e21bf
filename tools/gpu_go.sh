#!/bin/bash
# Build in-tree, then (only if the build succeeded) run the given command on the B200 via gpurun.
# Usage: tools/gpu_go.sh TIMEOUT 'command'
cd /root/repo
if ! python -c "from paper_1701_00182_b200 import build; build.build()" > /tmp/build.log 2>&1; then
  grep -iE "error" /tmp/build.log | head -20; echo BUILD FAILED; exit 1
fi
timeout $(( $1 + 1200 )) /usr/local/graft/bin/gpurun --timeout $1 -- "$2" 2>&1 | tail -2
