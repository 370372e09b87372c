#!/bin/bash
# One ncu capture (source counters + stall/pipe sections) of the kernel matching REGEX,
# after the same bench command exited 0 without ncu.
#   gpurun --timeout 1500 -- 'bash tools/gpu_prof_k.sh TAG REGEX [bench args...]'
set -u
TAG=$1; RX=$2; shift 2
mkdir -p gpurun_out
CMD="python bench.py --steps 2 --warmup 1 --no-net $*"
timeout 600 $CMD > gpurun_out/plain_$TAG.log 2>&1
RC=$?
echo "plain exit $RC" >> gpurun_out/plain_$TAG.log
if [ "$RC" = "0" ]; then
  timeout 900 ncu --section SourceCounters --section WarpStateStats --section InstructionStats \
      --section ComputeWorkloadAnalysis --section MemoryWorkloadAnalysis --section SpeedOfLight \
      --section Occupancy --section LaunchStats --section SchedulerStats \
      --metrics dram__bytes_read.sum,dram__bytes_write.sum,l1tex__data_pipe_lsu_wavefronts_mem_shared.sum,smsp__sass_thread_inst_executed_op_dadd_pred_on.sum,smsp__sass_thread_inst_executed_op_dmul_pred_on.sum,smsp__sass_thread_inst_executed_op_dfma_pred_on.sum \
      --clock-control none --import-source on -k regex:"$RX" -s 1 -c 1 \
      -o gpurun_out/prof_$TAG -f $CMD > gpurun_out/ncu_$TAG.log 2>&1
  echo "ncu exit $?" >> gpurun_out/ncu_$TAG.log
fi
exit 0
