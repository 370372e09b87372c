#!/bin/bash
# Quick GPU iteration: parity tests + bench for each BR lanes-per-CTA setting,
# optional ncu full capture of the blind-rotation kernel (after a clean run).
#   gpurun --timeout 1800 -- 'bash tools/gpu_quick.sh TAG [ncu]'
set -u
TAG=${1:-q}
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q -p no:cacheprovider > gpurun_out/pytest_gpu_$TAG.log 2>&1
echo "pytest exit $?" >> gpurun_out/pytest_gpu_$TAG.log
for G in 4 5; do
  SHE_BR_LANES_PER_CTA=$G timeout 600 python bench.py --steps 3 --warmup 3 > gpurun_out/bench_${TAG}_G$G.log 2>&1
  echo "bench exit $?" >> gpurun_out/bench_${TAG}_G$G.log
done
if [ "${2:-}" = "ncu" ]; then
  CMD="python bench.py --steps 2 --warmup 1"
  SHE_BR_LANES_PER_CTA=4 timeout 600 $CMD > gpurun_out/plain_$TAG.log 2>&1 && \
  SHE_BR_LANES_PER_CTA=4 timeout 900 ncu --set full --clock-control none --import-source on -k regex:br_kernel -s 1 -c 1 \
      -o gpurun_out/prof_br_$TAG -f $CMD > gpurun_out/ncu_full_$TAG.log 2>&1
  echo "ncu exit $?" >> gpurun_out/ncu_full_$TAG.log
fi
exit 0
