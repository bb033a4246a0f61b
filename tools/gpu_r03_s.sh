#!/bin/bash
# partition prefetch by bulk copies for int32 only; apply pair fetch by bulk copies (int32 / both / none)
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { cat gpurun_out/build.log; exit 1; }
timeout 900 python -m pytest tests/test_gpu_parity.py -q -m gpu -x -k "scatter" > gpurun_out/tests_s.log 2>&1; tail -2 gpurun_out/tests_s.log
VARIANTS="prev:@variants/libjacc.prev.so abulk2:-DSA_BULK=2 abulk0:-DSA_BULK=0" LOOPS="scat_f64 scat_i32" REPS=8 ROUNDS=2 bash tools/variant_ab.sh 2>&1 | tee gpurun_out/scat_ab_s.log
