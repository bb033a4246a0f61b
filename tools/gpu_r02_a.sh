#!/bin/bash
# round-2 first call: GPU tests after the advisor fixes, binned-scatter stress
# loop, RED throughput probe, sanitizers over every shared-memory kernel
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { cat gpurun_out/build.log; exit 1; }
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/gpu.txt
timeout 1500 python -m pytest tests -q -m gpu -x --timeout 600 > gpurun_out/gpu_tests.log 2>&1
tail -5 gpurun_out/gpu_tests.log
timeout 900 python tools/stress_scatter.py 200 i32_1 f64_1 i32_3 f64_2 > gpurun_out/stress_small.jsonl 2> gpurun_out/stress_small.err
timeout 900 python tools/stress_scatter.py 25 full_f64 full_i32 > gpurun_out/stress_full.jsonl 2> gpurun_out/stress_full.err
cat gpurun_out/stress_*.jsonl; tail -3 gpurun_out/stress_small.err
nvcc -O3 -gencode arch=compute_100a,code=sm_100a -o /tmp/red_probe tools/red_probe.cu && timeout 300 /tmp/red_probe > gpurun_out/red_probe.txt 2>&1
bash tools/gpu_sanitize.sh
