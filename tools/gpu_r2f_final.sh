#!/bin/bash
# Round-2f measurement call (TMEM engine, chunk queue by default, no L2 persisting window): smoke, GPU suite, the default bench (net,
# leveled units), the TCN / DSHE nets, then ncu: the launch list of the
# no-net bench and one capture each of the blind rotation and the tcgen05 key
# switch (ncu only after the same command exited 0 without it).
#   gpurun --timeout 3000 -- 'bash tools/gpu_r2f_final.sh TAG'
set -u
TAG=${1:-final}
mkdir -p gpurun_out
nvidia-smi -L > gpurun_out/smi_$TAG.txt 2>&1
nproc > gpurun_out/nproc_$TAG.txt
timeout 600 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_$TAG.log 2>&1
echo "smoke exit $?" >> gpurun_out/smoke_$TAG.log
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider -rf > gpurun_out/pytest_gpu_$TAG.log 2>&1
echo "pytest exit $?" >> gpurun_out/pytest_gpu_$TAG.log
timeout 900 python bench.py --steps 5 --warmup 3 > gpurun_out/bench_$TAG.log 2>&1
echo "bench exit $?" >> gpurun_out/bench_$TAG.log
timeout 1200 python bench.py --steps 3 --warmup 3 --tcn --dshe > gpurun_out/bench_nets_$TAG.log 2>&1
echo "bench nets exit $?" >> gpurun_out/bench_nets_$TAG.log
CMD="python bench.py --steps 2 --warmup 1 --no-net"
timeout 600 $CMD > gpurun_out/plain_$TAG.log 2>&1
RC=$?
echo "plain exit $RC" >> gpurun_out/plain_$TAG.log
if [ "$RC" = "0" ]; then
  timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 120 --csv \
      --log-file gpurun_out/launches_$TAG.csv $CMD > gpurun_out/ncu_launches_$TAG.log 2>&1
  echo "ncu launches exit $?" >> gpurun_out/ncu_launches_$TAG.log
  timeout 900 ncu --section SourceCounters --section WarpStateStats --section InstructionStats \
      --section ComputeWorkloadAnalysis --section MemoryWorkloadAnalysis --section SpeedOfLight \
      --section Occupancy --section LaunchStats --section SchedulerStats \
      --metrics dram__bytes_read.sum,dram__bytes_write.sum,smsp__sass_thread_inst_executed_op_dadd_pred_on.sum,smsp__sass_thread_inst_executed_op_dmul_pred_on.sum,smsp__sass_thread_inst_executed_op_dfma_pred_on.sum \
      --clock-control none --import-source on -k regex:"br_fft_tm_kernel" -s 1 -c 1 \
      -o gpurun_out/prof_fft_$TAG -f $CMD > gpurun_out/ncu_fft_$TAG.log 2>&1
  echo "ncu fft exit $?" >> gpurun_out/ncu_fft_$TAG.log
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:"ksi_gemm_tc" -s 1 -c 1 \
      -o gpurun_out/prof_ks_$TAG -f $CMD > gpurun_out/ncu_ks_$TAG.log 2>&1
  echo "ncu ks exit $?" >> gpurun_out/ncu_ks_$TAG.log
  # text exports for profiles/ (the .ncu-rep files stay in gpurun_out/)
  ncu -i gpurun_out/prof_fft_$TAG.ncu-rep --page raw --csv > gpurun_out/ncu_br_fft_tm_kernel_${TAG}_raw.csv 2>/dev/null
  ncu -i gpurun_out/prof_fft_$TAG.ncu-rep --page details --csv > gpurun_out/ncu_br_fft_tm_kernel_${TAG}_details.csv 2>/dev/null
  ncu -i gpurun_out/prof_ks_$TAG.ncu-rep --page details --csv > gpurun_out/ncu_ksi_gemm_tc_${TAG}_details.csv 2>/dev/null
fi
exit 0
