#!/bin/bash
# Time km_tc_filter_kernel (ncu launch list) and the C5 Lloyd loop for the default build and each variant.
for v in default build/variants/*/; do
  lib=""; [ "$v" != default ] && lib=$PWD/$v/libsketchcu.so
  SKC_LIB=$lib ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/ab.csv \
    -k regex:km_tc_filter timeout 300 python tools/kmeans_iters.py c5 3 > /dev/null 2>&1
  echo "$v filter: $(python tools/launch_seq.py gpurun_out/ab.csv km_tc_f | tail -1)"
  SKC_LIB=$lib timeout 300 python tools/kmeans_iters.py c5 | tail -1
done
