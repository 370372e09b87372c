#!/bin/bash
# Quick GPU iteration: parity tests + bench for each blind-rotation launch
# shape (SHE_BR_CFG=GxB), optional ncu full capture of the default shape.
#   gpurun --timeout 1800 -- 'bash tools/gpu_quick.sh TAG [ncu] [cfgs...]'
set -u
TAG=${1:-q}; NCU=${2:-}; shift 2 || shift $#
CFGS=${*:-"5x1 4x1 3x1 2x2 1x4"}
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q -p no:cacheprovider > gpurun_out/pytest_gpu_$TAG.log 2>&1
echo "pytest exit $?" >> gpurun_out/pytest_gpu_$TAG.log
for C in $CFGS; do
  SHE_BR_CFG=$C timeout 600 python bench.py --steps 3 --warmup 3 > gpurun_out/bench_${TAG}_$C.log 2>&1
  echo "bench exit $?" >> gpurun_out/bench_${TAG}_$C.log
done
if [ "$NCU" = "ncu" ]; then
  CMD="python bench.py --steps 2 --warmup 1"
  timeout 600 $CMD > gpurun_out/plain_$TAG.log 2>&1 && \
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:br_kernel -s 1 -c 1 \
      -o gpurun_out/prof_br_$TAG -f $CMD > gpurun_out/ncu_full_$TAG.log 2>&1
  echo "ncu exit $?" >> gpurun_out/ncu_full_$TAG.log
fi
exit 0
