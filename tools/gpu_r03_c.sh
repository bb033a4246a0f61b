#!/bin/bash
# dirty bits set by the apply (RED.OR) vs the bits pass; ncu --set full of the partition and apply
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { cat gpurun_out/build.log; exit 1; }
VARIANTS="bitsred:-DSA_BITS_RED=1 pfb1:-DSA_PFB=1" LOOPS="scat_f64 scat_i32" REPS=8 ROUNDS=2 bash tools/variant_ab.sh 2>&1 | tee gpurun_out/scat_ab_c.log
timeout 600 ncu --set full --import-source on --clock-control none -k regex:"scat_part_pf|scat_apply|scat_bits" -c 3 -o gpurun_out/scat_full_r03 python tools/ncu_target.py scatter 1 > gpurun_out/ncu_c.log 2>&1
tail -3 gpurun_out/ncu_c.log
