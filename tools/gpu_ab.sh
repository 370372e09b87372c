#!/bin/bash
# A/B of blind-rotation launch shapes: GPU parity tests under the first shape,
# then a bench line (no net) per shape.
#   gpurun -- 'bash tools/gpu_ab.sh TAG shape1 [shape2 ...]'
set -u
TAG=$1; shift
mkdir -p gpurun_out
SHE_BR_CFG=$1 timeout 900 python -m pytest tests -m gpu -x -q -p no:cacheprovider > gpurun_out/pytest_gpu_$TAG.log 2>&1
echo "pytest ($1) exit $?" >> gpurun_out/pytest_gpu_$TAG.log
for C in "$@"; do
  SHE_BR_CFG=$C timeout 600 python bench.py --steps 3 --warmup 3 --no-net > gpurun_out/bench_${TAG}_$C.log 2>&1
  echo "bench exit $?" >> gpurun_out/bench_${TAG}_$C.log
done
exit 0
