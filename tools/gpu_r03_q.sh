#!/bin/bash
# bulk range merge + Himeno bulk copy rows-per-warp: parity and A/B
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { cat gpurun_out/build.log; exit 1; }
timeout 1500 python -m pytest tests -q -m gpu -x -k "himeno or eager or jacobi or gemm or graph or random_programs or multiprocess or fig4 or square" > gpurun_out/tests_q.log 2>&1; tail -2 gpurun_out/tests_q.log
VARIANTS="rpw4:-DHIMENO_CB_RPW=4 rpw16:-DHIMENO_CB_RPW=16 rpw2:-DHIMENO_CB_RPW=2" LOOPS="himeno_copy" REPS=20 ROUNDS=2 bash tools/variant_ab.sh 2>&1 | tee gpurun_out/him_ab_q.log
LIB=paper_2110_14340_b200/libjacc.so; cp $LIB /tmp/new.so
for r in 1 2; do
  cp /tmp/new.so $LIB; echo -n "new "; timeout 600 python tools/merge_time.py 2>/dev/null | tail -1
  cp variants/libjacc.prev.so $LIB; echo -n "prev "; timeout 600 python tools/merge_time.py 2>/dev/null | tail -1
done | tee gpurun_out/merge_ab_q.log
cp /tmp/new.so $LIB
