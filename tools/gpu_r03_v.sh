#!/bin/bash
# Jacobi full-band fast path: parity + A/B + instruction count
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { cat gpurun_out/build.log; exit 1; }
timeout 1500 python -m pytest tests -q -m gpu -x -k "jacobi or J256 or J16K or halo or eager or smoke or graph or multiprocess" > gpurun_out/tests_v.log 2>&1; tail -2 gpurun_out/tests_v.log
VARIANTS="prev:@variants/libjacc.prev.so" LOOPS="jacobi" REPS=50 ROUNDS=3 bash tools/variant_ab.sh 2>&1 | tee gpurun_out/jac_ab_v.log
timeout 600 ncu --metrics gpu__time_duration.sum,smsp__inst_executed.sum,dram__bytes_read.sum,sm__inst_issued.avg.pct_of_peak_sustained_active --clock-control none -k regex:jacobi2d -c 2 --csv python tools/ncu_target.py jacobi 1 2>/dev/null | grep jacobi2d | awk -F'","' '{print $(NF-2), $NF}' | tail -4
