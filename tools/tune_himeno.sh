#!/bin/bash
# Himeno XL stencil variants: ncu launch durations
for v in ${VARIANTS:-0 1}; do
  JACC_HIMENO_VARIANT=$v timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum --clock-control none -k "regex:himeno_(stencil|march)" --csv --log-file gpurun_out/himeno_v$v.csv python tools/ncu_target.py himeno 2 > /dev/null 2>&1
  echo "variant $v"; grep -E "gpu__time|dram" gpurun_out/himeno_v$v.csv | awk -F'","' '{print $(NF-2), $NF}'
done
