#!/bin/bash
# One gpurun call: smoke, GPU parity tests, bench, then ncu (launch list + one
# full capture of the blind-rotation kernel) — ncu only after the same bench
# command exited 0 without it (B200_PROFILING.md).
#   gpurun --timeout 2400 -- 'bash tools/gpu_round.sh [tag] [ncu]'
set -u
TAG=${1:-r}
NCU=${2:-ncu}
mkdir -p gpurun_out
nvidia-smi -L > gpurun_out/smi_$TAG.txt 2>&1
nproc > gpurun_out/nproc_$TAG.txt; lscpu | head -20 >> gpurun_out/nproc_$TAG.txt
timeout 600 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_$TAG.log 2>&1
echo "smoke exit $?" >> gpurun_out/smoke_$TAG.log
timeout 1200 python -m pytest tests -m gpu -x -q -p no:cacheprovider > gpurun_out/pytest_gpu_$TAG.log 2>&1
echo "pytest exit $?" >> gpurun_out/pytest_gpu_$TAG.log
CMD="python bench.py --steps 3 --warmup 3"
timeout 900 $CMD > gpurun_out/bench_$TAG.log 2>&1
RC=$?
echo "bench exit $RC" >> gpurun_out/bench_$TAG.log
if [ "$RC" = "0" ] && [ "$NCU" = "ncu" ]; then
  timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 60 --csv \
      --log-file gpurun_out/launches_$TAG.csv $CMD > gpurun_out/ncu_launches_$TAG.log 2>&1
  echo "ncu launches exit $?" >> gpurun_out/ncu_launches_$TAG.log
  timeout 1200 ncu --set full --clock-control none --import-source on -k regex:br_kernel -s 1 -c 1 \
      -o gpurun_out/prof_br_$TAG -f $CMD > gpurun_out/ncu_full_$TAG.log 2>&1
  echo "ncu full exit $?" >> gpurun_out/ncu_full_$TAG.log
fi
exit 0
