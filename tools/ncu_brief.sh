#!/bin/bash
# ncu --set full of one kernel, summarised on the box (details page + top
# stall reasons per source line), report deleted unless KEEP=1
#   tools/ncu_brief.sh <tag> <kernel-regex> <skip> <cmd...>
tag=$1; k=$2; skip=$3; shift 3
timeout 900 ncu --set full --clock-control none --import-source on -k regex:$k -s $skip -c 1 -f -o gpurun_out/prof_$tag "$@" > gpurun_out/ncu_$tag.log 2>&1
ncu -i gpurun_out/prof_$tag.ncu-rep --page details --csv > gpurun_out/ncu_${tag}_details.csv 2>/dev/null
ncu -i gpurun_out/prof_$tag.ncu-rep --page raw --csv > gpurun_out/ncu_${tag}_raw.csv 2>/dev/null
ncu -i gpurun_out/prof_$tag.ncu-rep --page source --csv > gpurun_out/ncu_${tag}_source.csv 2>/dev/null
[ "${KEEP:-0}" = 1 ] || rm -f gpurun_out/prof_$tag.ncu-rep
ls -la gpurun_out/ncu_${tag}_*.csv | awk '{print $5, $9}'
