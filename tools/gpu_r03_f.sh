#!/bin/bash
# Jacobi band interleave vs previous build; Himeno cache-policy / copy-shape variants; parity
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { cat gpurun_out/build.log; exit 1; }
timeout 1200 python -m pytest tests -q -m gpu -x -k "jacobi or multiprocess or smoke or halo or himeno" > gpurun_out/tests_f.log 2>&1; tail -2 gpurun_out/tests_f.log
VARIANTS="prev:@variants/libjacc.prev.so nobw:-DJACC_JACOBI_BW=0" LOOPS="jacobi" REPS=50 ROUNDS=3 bash tools/variant_ab.sh 2>&1 | tee gpurun_out/jac_ab_f.log
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:jacobi2d -c 4 --csv python tools/ncu_target.py jacobi 2 2>/dev/null | grep jacobi2d | awk -F'","' '{print $(NF-2), $NF}' | tail -6
VARIANTS="pl2:-DHIMENO_PL2=1 cef:-DHIMENO_CEF=1 pl2cef:-DHIMENO_PL2=1,-DHIMENO_CEF=1 cm3:-DHIMENO_COPY_MINB=3 cm4h1:-DHIMENO_COPY_MINB=4,-DHIMENO_HC=1 cg2:-DHIMENO_COPY_GRID=2 cm3g3:-DHIMENO_COPY_MINB=3,-DHIMENO_COPY_GRID=3" LOOPS="himeno himeno_copy" REPS=10 ROUNDS=2 bash tools/variant_ab.sh 2>&1 | tee gpurun_out/him_ab_f.log
