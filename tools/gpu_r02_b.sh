#!/bin/bash
# round-2 call b: new parity tests, the restructured bench (both arms)
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { cat gpurun_out/build.log; exit 1; }
timeout 1500 python -m pytest tests/test_gpu_parity.py -q -m gpu --timeout 900 -k "add_order or random_field or 200_launches or uniform_tolerance or regrowth or in_capture or back_to_back or inactive or cross_device_same_queue" > gpurun_out/gpu_tests_b.log 2>&1
tail -5 gpurun_out/gpu_tests_b.log
timeout 1200 python bench.py > gpurun_out/bench_b.json 2> gpurun_out/bench_b.err
tail -3 gpurun_out/bench_b.err
timeout 600 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/bench_ref_b.json 2> gpurun_out/bench_ref_b.err
cat gpurun_out/bench_ref_b.json; tail -3 gpurun_out/bench_ref_b.err
