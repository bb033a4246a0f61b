#!/bin/bash
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { cat gpurun_out/build.log; exit 1; }
timeout 1200 python -m pytest tests/test_gpu_parity.py -q -m gpu --timeout 600 -k "fig4 or himeno or nccl or trace or info" > gpurun_out/gpu_tests_j.log 2>&1
tail -3 gpurun_out/gpu_tests_j.log
bash tools/gpu_sanitize.sh
grep -A6 "hazard detected" gpurun_out/san_racecheck_r02.log | grep -oE "Host Frame: jk::[a-z_0-9]+|in kernels.cu:[0-9]+" | sort | uniq -c | sort -rn | head
