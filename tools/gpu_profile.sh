#!/bin/bash
# Round profile: full bench (with net latency), ncu launch list of the bench
# command, one ncu --set full capture each of the BR and KS kernels.
#   gpurun --timeout 2400 -- 'bash tools/gpu_profile.sh TAG'
set -u
TAG=${1:-p}
mkdir -p gpurun_out
nvidia-smi -L > gpurun_out/smi_$TAG.txt 2>&1
timeout 1200 python bench.py --steps 5 --warmup 3 > gpurun_out/bench_$TAG.log 2>&1
echo "bench exit $?" >> gpurun_out/bench_$TAG.log
CMD="python bench.py --steps 2 --warmup 1 --no-net"
timeout 600 $CMD > gpurun_out/plain_$TAG.log 2>&1 && \
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 60 --csv \
    --log-file gpurun_out/launches_$TAG.csv $CMD > gpurun_out/ncu_launches_$TAG.log 2>&1
echo "ncu launches exit $?" >> gpurun_out/ncu_launches_$TAG.log
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:"br_(fft_)?kernel" -s 1 -c 1 \
    -o gpurun_out/prof_br_$TAG -f $CMD > gpurun_out/ncu_br_$TAG.log 2>&1
echo "ncu br exit $?" >> gpurun_out/ncu_br_$TAG.log
timeout 900 ncu --set full --clock-control none --import-source on -k regex:ks2_kernel -s 1 -c 1 \
    -o gpurun_out/prof_ks_$TAG -f $CMD > gpurun_out/ncu_ks_$TAG.log 2>&1
echo "ncu ks exit $?" >> gpurun_out/ncu_ks_$TAG.log
exit 0
