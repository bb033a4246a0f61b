#!/bin/bash
# compute-sanitizer memcheck / racecheck over small parity cases
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
K='J256 or test_jacobi_multi_device and 17- or test_scatter_exact and 100- or test_square_multi and 1000- or test_dot_sum_dyadic_exact and 4096 or test_gemm_random_tolerance and 37 or himeno_multi_device and shape1 or fig4_chain and -257- or iteration_split and 100003 and f64 or test_graph_capture or async_queues'
timeout 1500 compute-sanitizer --tool memcheck --leak-check no --error-exitcode 9 python -m pytest tests/test_gpu_parity.py -q -m gpu -k "$K" > gpurun_out/memcheck.log 2>&1; echo "memcheck rc=$?" >> gpurun_out/memcheck.log
timeout 1500 compute-sanitizer --tool racecheck --error-exitcode 9 python -m pytest tests/test_gpu_parity.py -q -m gpu -k "J256 or test_scatter_exact and 100-" > gpurun_out/racecheck.log 2>&1; echo "racecheck rc=$?" >> gpurun_out/racecheck.log
tail -4 gpurun_out/memcheck.log; tail -4 gpurun_out/racecheck.log
