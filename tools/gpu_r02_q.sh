#!/bin/bash
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || exit 1
for r in 1 2; do for l in scat_f64 scat_i32; do timeout 300 python tools/time_loop.py $l 8; done; done
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:scat_apply --csv python tools/ncu_target.py scatter 2 2>/dev/null | grep scat_apply | tail -2 | awk -F'","' '{print $(NF-2), $NF}'
timeout 900 python -m pytest tests/test_gpu_parity.py -q -m gpu -x -k "scatter" 2>&1 | tail -2
timeout 600 python tools/stress_scatter.py 10 i32_1 f64_2 full_f64 full_i32
