#!/bin/bash
# plane-marching Himeno stencil: parity, A/B vs the row-per-warp kernel, DRAM bytes
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { cat gpurun_out/build.log; exit 1; }
timeout 1500 python -m pytest tests -q -m gpu -x -k "himeno" > gpurun_out/tests_h.log 2>&1; tail -2 gpurun_out/tests_h.log
VARIANTS="prev:@variants/libjacc.prev.so" LOOPS="himeno" REPS=10 ROUNDS=3 bash tools/variant_ab.sh 2>&1 | tee gpurun_out/him_ab_h.log
M="gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sector_hit_rate.pct"
timeout 600 ncu --metrics $M --clock-control none -k regex:himeno_stencil -c 2 --csv python tools/ncu_target.py himeno 2 2>/dev/null | grep himeno_stencil | awk -F'","' '{print $(NF-2), $NF}' | tail -4
