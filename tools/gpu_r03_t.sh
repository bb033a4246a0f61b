#!/bin/bash
# bits pass: key batch made a control dependency of its atomics; parity + A/B
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { cat gpurun_out/build.log; exit 1; }
timeout 900 python -m pytest tests/test_gpu_parity.py -q -m gpu -x -k "scatter" > gpurun_out/tests_t.log 2>&1; tail -2 gpurun_out/tests_t.log
VARIANTS="prev:@variants/libjacc.prev.so" LOOPS="scat_f64 scat_i32" REPS=8 ROUNDS=3 bash tools/variant_ab.sh 2>&1 | tee gpurun_out/scat_ab_t.log
for w in scatter scatter_i32; do timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:scat_bits --csv python tools/ncu_target.py $w 2 2>/dev/null | grep scat_bits | awk -F'","' '{print $NF}' | tail -1; done
