#!/bin/bash
# A/B of library variants built by tools/build_variant.sh into varbuild/:
# each NAME.so is swapped in as libshe.so for one config-1 bench (plain run).
#   gpurun --timeout 1500 -- 'bash tools/gpu_var.sh TAG name1 name2 ...'
set -u
TAG=$1; shift
mkdir -p gpurun_out
L=paper_1906_00148_b200/libshe.so
cp $L /tmp/libshe_default.so
for V in default "$@"; do
  if [ "$V" = "default" ]; then cp /tmp/libshe_default.so $L; else cp varbuild/$V.so $L; fi
  touch $L
  timeout 600 python bench.py --no-net --steps 5 --warmup 3 > gpurun_out/var_${TAG}_$V.log 2>&1
  echo "exit $?" >> gpurun_out/var_${TAG}_$V.log
done
cp /tmp/libshe_default.so $L
exit 0
