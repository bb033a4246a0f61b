#!/bin/bash
# flat-chunk Himeno copy: parity and shape variants vs the row-per-warp copy
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { cat gpurun_out/build.log; exit 1; }
timeout 1500 python -m pytest tests -q -m gpu -x -k "himeno" > gpurun_out/tests_i.log 2>&1; tail -2 gpurun_out/tests_i.log
VARIANTS="rows:-DHIMENO_COPY_FLAT=0 g4:-DHIMENO_COPY_GRID=4 g16:-DHIMENO_COPY_GRID=16 u8:-DHIMENO_HCU=8 u2g16:-DHIMENO_HCU=2,-DHIMENO_COPY_GRID=16" LOOPS="himeno_copy" REPS=20 ROUNDS=2 bash tools/variant_ab.sh 2>&1 | tee gpurun_out/him_ab_i.log
M="gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum"
timeout 600 ncu --metrics $M --clock-control none -k regex:himeno_copy -c 2 --csv python tools/ncu_target.py himeno 2 2>/dev/null | grep himeno_copy | awk -F'","' '{print $(NF-2), $NF}' | tail -3
