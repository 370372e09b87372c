#!/bin/bash
# FFT engine A/B: gate parity tests, then bench.py --no-net per shape
mkdir -p gpurun_out
TAG=${1:-t}
timeout 600 python -m pytest tests/test_gpu_gates.py -x -q -p no:cacheprovider > gpurun_out/fft_gates_$TAG.log 2>&1; echo "exit $?" >> gpurun_out/fft_gates_$TAG.log
for e in ${ENGINES:-fft3 fft4 fft5}; do SHE_BR_ENGINE=$e timeout 300 python bench.py --no-net --steps 5 --warmup 3 > gpurun_out/fft_bench_${e}_$TAG.log 2>&1; done
