mkdir -p gpurun_out
export SHE_BR_ENGINE=fft
timeout 600 python -m pytest tests/test_gpu_gates.py -x -q -p no:cacheprovider > gpurun_out/fft_gates.log 2>&1; echo "exit $?" >> gpurun_out/fft_gates.log
for e in fft4 fft3; do SHE_BR_ENGINE=$e timeout 300 python bench.py --no-net --steps 3 --warmup 3 > gpurun_out/fft_bench_$e.log 2>&1; done
