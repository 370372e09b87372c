#!/bin/bash
# A/B build of libshe.so with extra -D flags into OUT (experiments only; the
# product build is paper_1906_00148_b200/build.py):
#   bash tools/build_variant.sh OUT.so -DSHE_TM_PD=2 ...
set -e
OUT=$1; shift
D=$(cd "$(dirname "$0")/.." && pwd)/paper_1906_00148_b200/csrc
T=$(mktemp -d)
FL="-gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -lineinfo --expt-relaxed-constexpr -DGL_ADDSUB_PTX -Xcompiler -fPIC,-fopenmp,-ffp-contract=off,-march=x86-64-v3"
nvcc $FL "$@" -c $D/engine.cu -o $T/engine.o
nvcc $FL -c $D/client.cpp -o $T/client.o
nvcc $FL -c $D/scheduler.cpp -o $T/scheduler.o
nvcc -gencode arch=compute_100a,code=sm_100a -shared -Xcompiler -fPIC,-fopenmp $T/*.o -o "$OUT" -lcudart -lgomp
rm -rf $T
