#!/bin/bash
# Jacobi with alternating band directions vs previous build; parity; mp info
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { cat gpurun_out/build.log; exit 1; }
timeout 1200 python -m pytest tests -q -m gpu -x -k "jacobi or multiprocess or smoke or halo or eager" > gpurun_out/tests_e.log 2>&1; tail -2 gpurun_out/tests_e.log
VARIANTS="prev:@variants/libjacc.prev.so" LOOPS="jacobi" REPS=50 ROUNDS=3 bash tools/variant_ab.sh 2>&1 | tee gpurun_out/jac_ab_e.log
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:jacobi2d -c 6 --csv python tools/ncu_target.py jacobi 3 2>/dev/null | grep jacobi2d | awk -F'","' '{print $(NF-2), $NF}' | tail -12
