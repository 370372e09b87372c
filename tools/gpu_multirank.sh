#!/bin/bash
# Functional check of the N > 1 bench path on ONE GPU: 2 ranks over gloo, both
# on device 0 (no kernel waits on another rank; timings are meaningless).
#   gpurun -- 'bash tools/gpu_multirank.sh TAG'
set -u
TAG=${1:-mr}
mkdir -p gpurun_out
SHE_BENCH_BACKEND=gloo SHE_BENCH_DEVICE=0 timeout 1200 python -m torch.distributed.run --nnodes=1 \
    --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29512 bench.py --gpus 2 --steps 2 \
    --warmup 1 > gpurun_out/bench_$TAG.log 2>&1
echo "bench exit $?" >> gpurun_out/bench_$TAG.log
exit 0
