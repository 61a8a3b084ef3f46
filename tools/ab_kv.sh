#!/bin/bash
# Time km_tc_verify_kernel (ncu launch list, 3rd launch) and the C5 Lloyd loop for the default build and each variant.
for v in default build/variants/*/; do
  lib=""; [ "$v" != default ] && lib=$PWD/$v/libsketchcu.so
  SKC_LIB=$lib ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/ab.csv \
    -k regex:${KREGEX:-km_tc_verify} timeout 300 python tools/kmeans_iters.py c5 4 > /dev/null 2>&1
  echo "$v: $(python tools/launch_seq.py gpurun_out/ab.csv ${KREGEX:-km_tc_verify} | tail -1)"
  SKC_LIB=$lib timeout 300 python tools/kmeans_iters.py c5 | tail -1
done
