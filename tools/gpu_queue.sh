#!/bin/bash
# Work-queue check of the TMEM engine: the gate-level GPU tests (config 0/1
# parity, every engine option, the queue's even/odd lane counts), then a
# config-1 bench per fft_chunk value (plain runs, no profiler).
#   gpurun --timeout 2400 -- 'bash tools/gpu_queue.sh TAG chunk...'
set -u
TAG=$1; shift
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_fft_selftest.py tests/test_gpu_gates.py -q -p no:cacheprovider -x \
    > gpurun_out/pytest_queue_$TAG.log 2>&1
echo "pytest exit $?" >> gpurun_out/pytest_queue_$TAG.log
for C in "$@"; do
  timeout 300 python bench.py --no-net --steps 5 --warmup 3 --fft-chunk $C > gpurun_out/queue_${TAG}_c$C.log 2>&1
  echo "exit $?" >> gpurun_out/queue_${TAG}_c$C.log
done
exit 0
