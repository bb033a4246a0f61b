#!/bin/bash
# Himeno copy by the bulk-copy engine: parity, A/B vs the row-per-warp copy
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { cat gpurun_out/build.log; exit 1; }
timeout 900 python -m pytest tests -q -m gpu -x -k "himeno" > gpurun_out/tests_n.log 2>&1; tail -2 gpurun_out/tests_n.log
VARIANTS="prev:@variants/libjacc.prev.so g4:-DHIMENO_CB_GRID=4 g16:-DHIMENO_CB_GRID=16 r8:-DHIMENO_CB_R=8,-DHIMENO_CB_GRID=4" LOOPS="himeno_copy" REPS=20 ROUNDS=2 bash tools/variant_ab.sh 2>&1 | tee gpurun_out/him_ab_n.log
