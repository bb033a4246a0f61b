#!/bin/bash
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { cat gpurun_out/build.log; exit 1; }
timeout 2400 python -m pytest tests -q -m gpu --timeout 900 > gpurun_out/gpu_tests_i.log 2>&1
tail -4 gpurun_out/gpu_tests_i.log
bash tools/gpu_sanitize.sh
timeout 600 python bench.py --gpus 2 --steps 2 --warmup 1 --no-cpu-baseline > gpurun_out/bench_sp2_loops.json 2> gpurun_out/bench_sp2_loops.err
tail -2 gpurun_out/bench_sp2_loops.err
