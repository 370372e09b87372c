#!/bin/bash
# A/B of the L2 persisting window over BK for the TMEM engine (the product
# library has none; varbuild/libshe_persist.so = tools/build_variant.sh with
# -DSHE_TM_PERSIST has it): config-1 bench and the blind rotation's DRAM bytes
# (ncu, one launch) for the chunk queue and the wrap-around schedule.
# (profiles/r2f/persist_ab.txt was taken when the window was still the default
# and the variant was the library without it.)
#   gpurun --timeout 1500 -- 'bash tools/gpu_persist.sh TAG'
set -u
TAG=$1
mkdir -p gpurun_out
L=paper_1906_00148_b200/libshe.so
cp $L /tmp/libshe_default.so
for V in default persist; do
  if [ "$V" = "default" ]; then cp /tmp/libshe_default.so $L; else cp varbuild/libshe_$V.so $L; fi
  touch $L
  for C in 0 -2; do
    CMD="python bench.py --no-net --steps 5 --warmup 3 --fft-chunk $C"
    timeout 300 $CMD > gpurun_out/persist_${TAG}_${V}_c$C.log 2>&1
    echo "exit $?" >> gpurun_out/persist_${TAG}_${V}_c$C.log
    timeout 300 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum,lts__t_sector_hit_rate.pct \
        --clock-control none -k regex:br_fft_tm_kernel -s 1 -c 1 --csv --log-file gpurun_out/persist_${TAG}_${V}_c$C.csv \
        $CMD > /dev/null 2>&1
  done
done
cp /tmp/libshe_default.so $L
exit 0
