#!/bin/bash
# Round profile of the FFT engine: GPU tests, bench (+ net), ncu launch list, one ncu --set full
# capture each of the BR and KS kernels, FP64 instruction counts, and the three nets.
#   gpurun --timeout 3000 -- "bash tools/gpu_fft_profile.sh TAG"
bash tools/gpu_tests.sh $1
bash tools/gpu_profile.sh $1
CMD="python bench.py --steps 2 --warmup 1 --no-net"
timeout 600 ncu --metrics smsp__sass_thread_inst_executed_op_dadd_pred_on.sum,smsp__sass_thread_inst_executed_op_dmul_pred_on.sum,smsp__sass_thread_inst_executed_op_dfma_pred_on.sum,sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active,sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active,smsp__issue_active.avg.pct_of_peak_sustained_active,l1tex__data_pipe_lsu_wavefronts_mem_shared.sum,sm__cycles_elapsed.avg --clock-control none -k regex:br_fft_kernel -s 1 -c 1 --csv $CMD > gpurun_out/ncu_fp64_$1.csv 2> gpurun_out/ncu_fp64_$1.err

timeout 1500 python bench.py --tcn --dshe --steps 3 --warmup 3 > gpurun_out/nets_$1.log 2>&1; echo "nets exit $?" >> gpurun_out/nets_$1.log
exit 0
