#!/bin/bash
# A/B of library variants with bench arguments: "name:variant:args" triples
# (variant = a varbuild/*.so, or "default").
#   gpurun --timeout 1500 -- 'bash tools/gpu_var2.sh TAG "a:indep:" "b:indep:--fft-stagger-ns 8000"'
set -u
TAG=$1; shift
mkdir -p gpurun_out
L=paper_1906_00148_b200/libshe.so
cp $L /tmp/libshe_default.so
for T in "$@"; do
  NAME=${T%%:*}; REST=${T#*:}; V=${REST%%:*}; ARGS=${REST#*:}
  if [ "$V" = "default" ]; then cp /tmp/libshe_default.so $L; else cp varbuild/$V.so $L; fi
  touch $L
  timeout 600 python bench.py --no-net --steps 5 --warmup 3 $ARGS > gpurun_out/var_${TAG}_$NAME.log 2>&1
  echo "exit $?" >> gpurun_out/var_${TAG}_$NAME.log
done
cp /tmp/libshe_default.so $L
exit 0
