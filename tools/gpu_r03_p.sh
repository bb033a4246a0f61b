#!/bin/bash
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { cat gpurun_out/build.log; exit 1; }
timeout 900 python -m pytest tests -q -m gpu -x -k "himeno" > gpurun_out/tests_p.log 2>&1; tail -2 gpurun_out/tests_p.log
VARIANTS="g48:-DHIMENO_CB_GRID=48 g64:-DHIMENO_CB_GRID=64 g128:-DHIMENO_CB_GRID=128 r6g48:-DHIMENO_CB_R=6,-DHIMENO_CB_GRID=48 r3g64:-DHIMENO_CB_R=3,-DHIMENO_CB_GRID=64" LOOPS="himeno_copy" REPS=20 ROUNDS=2 bash tools/variant_ab.sh 2>&1 | tee gpurun_out/him_ab_p.log
