#!/bin/bash
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || exit 1
for r in 1 2; do timeout 300 python tools/time_loop.py scat_f64 8; JACC_EXP_PART_T=128 timeout 300 python tools/time_loop.py scat_f64 8 | sed 's/^/T128 /'; done
JACC_EXP_PART_T=192 timeout 300 python tools/time_loop.py scat_f64 8 | sed "s/^/T192 /"
JACC_EXP_PART_T=128 timeout 300 python tools/stress_scatter.py 2 full_f64
