#!/bin/bash
# apply variants after the L2 prefetch; exact path with the prefetch; parity
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { cat gpurun_out/build.log; exit 1; }
timeout 900 python -m pytest tests/test_gpu_parity.py -q -m gpu -x -k "scatter" > gpurun_out/scat_tests_b.log 2>&1; tail -2 gpurun_out/scat_tests_b.log
for l in scat_f64 scat_i32; do echo -n "exact "; JACC_SCATTER_SPEC=0 timeout 300 python tools/time_loop.py $l 8; done | tee gpurun_out/scat_ab_b.log
VARIANTS="ch2k4:-DSA_CH=2048,-DSA_BPS=4 ch2k3:-DSA_CH=2048,-DSA_BPS=3 ch8k1:-DSA_CH=8192,-DSA_BPS=1 pf3ch2k4:-DSA_CH=2048,-DSA_BPS=4,-DSA_PFB=3 ch4k3i:-DSA_CH=4096,-DSA_BPS=3" \
LOOPS="scat_f64 scat_i32" REPS=8 ROUNDS=2 bash tools/variant_ab.sh 2>&1 | tee -a gpurun_out/scat_ab_b.log
