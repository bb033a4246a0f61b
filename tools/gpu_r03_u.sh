#!/bin/bash
# partition bulk prefetch for fp64, in pieces
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { cat gpurun_out/build.log; exit 1; }
VARIANTS="f64b:-DSCAT_PF_BULK_F64=1 f64p8k:-DSCAT_PF_BULK_F64=1,-DSCAT_PF_PIECE=8192u f64p4k:-DSCAT_PF_BULK_F64=1,-DSCAT_PF_PIECE=4096u f64p16k:-DSCAT_PF_BULK_F64=1,-DSCAT_PF_PIECE=16384u i32p8k:-DSCAT_PF_PIECE=8192u" LOOPS="scat_f64 scat_i32" REPS=8 ROUNDS=2 bash tools/variant_ab.sh 2>&1 | tee gpurun_out/scat_ab_u.log
