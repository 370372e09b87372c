#!/bin/bash
# A/B of the TMEM engine's grid for narrow batches: bench --sweep with the
# product library, then with varbuild/libshe_grid8.so (-DSHE_TM_GRID8) copied
# over it on the box's scratch copy.
#   gpurun --timeout 1500 -- 'bash tools/gpu_grid.sh TAG'
set -u
TAG=$1
mkdir -p gpurun_out
timeout 400 python bench.py --no-net --sweep --steps 3 --warmup 3 > gpurun_out/grid_${TAG}_new.log 2>&1
echo "exit $?" >> gpurun_out/grid_${TAG}_new.log
cp varbuild/libshe_grid8.so paper_1906_00148_b200/libshe.so
timeout 400 python bench.py --no-net --sweep --steps 3 --warmup 3 > gpurun_out/grid_${TAG}_grid8.log 2>&1
echo "exit $?" >> gpurun_out/grid_${TAG}_grid8.log
exit 0
