#!/bin/bash
# One compute-sanitizer tool per call (B200_PROFILING.md), after the plain run
# exited 0:  gpurun --timeout 1800 -- 'bash tools/gpu_sanitize.sh racecheck'
set -u
TOOL=${1:-racecheck}
mkdir -p gpurun_out
timeout 300 python tools/sanitize_small.py > gpurun_out/sanitize_plain.log 2>&1 && \
timeout 1500 compute-sanitizer --tool $TOOL --print-limit 50 python tools/sanitize_small.py \
    > gpurun_out/sanitize_$TOOL.log 2>&1
echo "exit $?" >> gpurun_out/sanitize_$TOOL.log
exit 0
