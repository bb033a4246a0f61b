#!/bin/bash
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { cat gpurun_out/build.log; exit 1; }
VARIANTS="g32:-DHIMENO_CB_GRID=32 r2g16:-DHIMENO_CB_R=2 r2g32:-DHIMENO_CB_R=2,-DHIMENO_CB_GRID=32 r3g24:-DHIMENO_CB_R=3,-DHIMENO_CB_GRID=24 g12:-DHIMENO_CB_GRID=12" LOOPS="himeno_copy" REPS=20 ROUNDS=2 bash tools/variant_ab.sh 2>&1 | tee gpurun_out/him_ab_o.log
