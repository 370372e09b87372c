#!/bin/bash
mkdir -p gpurun_out
TAG=${1:-m}
for V in 0 1; do timeout 120 ./tools/microbench/fb$V >> gpurun_out/micro_$TAG.log 2>&1; done
timeout 900 python -m pytest tests -m gpu -x -q -p no:cacheprovider > gpurun_out/pytest_gpu_$TAG.log 2>&1
echo "pytest exit $?" >> gpurun_out/pytest_gpu_$TAG.log
for G in 4 5; do
  SHE_BR_CFG=${G}x1 timeout 600 python bench.py --steps 3 --warmup 3 > gpurun_out/bench_${TAG}_G$G.log 2>&1
done
exit 0
