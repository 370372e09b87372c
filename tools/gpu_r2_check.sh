#!/bin/bash
# Round 2 functional check: full GPU suite (+ the FFT self-test with output),
# default bench, and the 2-rank bench over gloo on one GPU.
#   gpurun --timeout 2400 -- 'bash tools/gpu_r2_check.sh TAG'
set -u
TAG=${1:-c}
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -x -q -p no:cacheprovider -rA > gpurun_out/pytest_gpu_$TAG.log 2>&1
echo "pytest exit $?" >> gpurun_out/pytest_gpu_$TAG.log
timeout 300 python -m pytest tests/test_gpu_fft_selftest.py -q -s -p no:cacheprovider > gpurun_out/fft_selftest_$TAG.log 2>&1
timeout 600 python bench.py --steps 5 --warmup 3 > gpurun_out/bench_$TAG.log 2>&1
echo "bench exit $?" >> gpurun_out/bench_$TAG.log
SHE_BENCH_BACKEND=gloo timeout 600 python bench.py --gpus 2 --no-net --steps 3 --warmup 3 > gpurun_out/bench_gloo2_$TAG.log 2>&1
echo "bench gloo2 exit $?" >> gpurun_out/bench_gloo2_$TAG.log
exit 0
