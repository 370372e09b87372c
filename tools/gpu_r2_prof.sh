#!/bin/bash
# Round-2 profile of the blind-rotation kernel: plain bench (no net), then one
# ncu capture of br_fft_kernel with source-level stall counters (smaller than
# --set full so the report fits the gpurun_out merge limit).
#   gpurun --timeout 1500 -- 'bash tools/gpu_r2_prof.sh TAG [extra env]'
set -u
TAG=${1:-p}
mkdir -p gpurun_out
CMD="python bench.py --steps 2 --warmup 1 --no-net"
timeout 600 $CMD > gpurun_out/plain_$TAG.log 2>&1
RC=$?
echo "plain exit $RC" >> gpurun_out/plain_$TAG.log
if [ "$RC" = "0" ]; then
  timeout 900 ncu --section SourceCounters --section WarpStateStats --section InstructionStats \
      --section ComputeWorkloadAnalysis --section MemoryWorkloadAnalysis --section SpeedOfLight \
      --section Occupancy --section LaunchStats --section SchedulerStats \
      --clock-control none --import-source on -k regex:"br_fft_kernel" -s 1 -c 1 \
      -o gpurun_out/prof_fft_$TAG -f $CMD > gpurun_out/ncu_fft_$TAG.log 2>&1
  echo "ncu exit $?" >> gpurun_out/ncu_fft_$TAG.log
fi
ls -la gpurun_out/ > gpurun_out/ls_$TAG.txt
exit 0
