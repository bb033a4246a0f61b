#!/bin/bash
# partition phases with loads batched ahead of stores vs previous build; parity
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { cat gpurun_out/build.log; exit 1; }
timeout 900 python -m pytest tests/test_gpu_parity.py -q -m gpu -x -k "scatter" > gpurun_out/scat_tests_d.log 2>&1; tail -2 gpurun_out/scat_tests_d.log
VARIANTS="prev:@variants/libjacc.prev.so" LOOPS="scat_f64 scat_i32" REPS=8 ROUNDS=2 bash tools/variant_ab.sh 2>&1 | tee gpurun_out/scat_ab_d.log
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv python tools/ncu_target.py scatter 2 2>/dev/null | grep scat_ | awk -F'","' '{print $5, $NF}' | cut -c1-60,200- | tail -8
