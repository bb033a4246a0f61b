#!/bin/bash
# bits pass with batched key loads vs previous build; scatter parity
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { cat gpurun_out/build.log; exit 1; }
timeout 900 python -m pytest tests/test_gpu_parity.py -q -m gpu -x -k "scatter" > gpurun_out/tests_j.log 2>&1; tail -2 gpurun_out/tests_j.log
VARIANTS="prev:@variants/libjacc.prev.so u8:-DSBITS_U=8 u2:-DSBITS_U=2" LOOPS="scat_f64 scat_i32" REPS=8 ROUNDS=2 bash tools/variant_ab.sh 2>&1 | tee gpurun_out/bits_ab_j.log
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:scat_bits --csv python tools/ncu_target.py scatter 2 2>/dev/null | grep scat_bits | awk -F'","' '{print $NF}' | tail -2
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:scat_bits --csv python tools/ncu_target.py scatter_i32 2 2>/dev/null | grep scat_bits | awk -F'","' '{print $NF}' | tail -2
