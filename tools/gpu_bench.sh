#!/bin/bash
# Full bench (gates/s + net latency) then ncu launch list and one full capture.
#   gpurun --timeout 2400 -- 'bash tools/gpu_bench.sh TAG [ncu]'
set -u
TAG=${1:-b}
mkdir -p gpurun_out
nproc > gpurun_out/nproc_$TAG.txt; lscpu | head -20 >> gpurun_out/nproc_$TAG.txt
timeout 1200 python bench.py --steps 5 --warmup 3 > gpurun_out/bench_$TAG.log 2>&1
echo "bench exit $?" >> gpurun_out/bench_$TAG.log
if [ "${2:-}" = "ncu" ]; then
  CMD="python bench.py --steps 2 --warmup 1 --no-net"
  timeout 600 $CMD > gpurun_out/plain_$TAG.log 2>&1 && \
  timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 60 --csv \
      --log-file gpurun_out/launches_$TAG.csv $CMD > gpurun_out/ncu_launches_$TAG.log 2>&1
  echo "ncu launches exit $?" >> gpurun_out/ncu_launches_$TAG.log
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:ks_kernel -s 1 -c 1 \
      -o gpurun_out/prof_ks_$TAG -f $CMD > gpurun_out/ncu_ks_$TAG.log 2>&1
  echo "ncu ks exit $?" >> gpurun_out/ncu_ks_$TAG.log
fi
exit 0
