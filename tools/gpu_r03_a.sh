#!/bin/bash
# speculative fixed-capacity scatter layout + L2 prefetch of a: parity and A/B timing
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { cat gpurun_out/build.log; exit 1; }
timeout 900 python -m pytest tests/test_gpu_parity.py -q -m gpu -x -k "scatter" > gpurun_out/scat_tests.log 2>&1; tail -3 gpurun_out/scat_tests.log
for r in 1 2; do
 for cfg in "0 0" "1 0" "1 2" "1 3" "1 1"; do
  set -- $cfg
  for l in scat_f64 scat_i32; do
   echo -n "spec=$1 pfb=$2 "; JACC_SCATTER_SPEC=$1 JACC_SCATTER_PFB=$2 timeout 300 python tools/time_loop.py $l 8
  done
 done
done 2>&1 | tee gpurun_out/scat_ab.log
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv python tools/ncu_target.py scatter 2 > gpurun_out/scat_ncu.csv 2>/dev/null
grep scat_ gpurun_out/scat_ncu.csv | awk -F'","' '{print $5, $(NF-2), $NF}' | tail -30
