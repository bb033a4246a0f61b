#!/bin/bash
# full validation + measurements of record after the late round-2 scatter changes
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { cat gpurun_out/build.log; exit 1; }
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; tail -1 gpurun_out/smoke.log
timeout 2400 python -m pytest tests -q -m gpu --timeout 900 > gpurun_out/gpu_tests_final.log 2>&1
tail -3 gpurun_out/gpu_tests_final.log
timeout 1200 python tools/stress_scatter.py 200 i32_1 f64_1 i32_3 f64_2 > gpurun_out/stress_final.jsonl 2> gpurun_out/stress_final.err
timeout 900 python tools/stress_scatter.py 25 full_f64 full_i32 >> gpurun_out/stress_final.jsonl 2>> gpurun_out/stress_final.err
tail -6 gpurun_out/stress_final.jsonl
ROUND_TAG=r02 bash tools/gpu_round.sh

