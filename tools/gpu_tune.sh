#!/bin/bash
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { cat gpurun_out/build.log; exit 1; }
timeout 900 python -m pytest tests -q -m gpu -x -k "not full_size" > gpurun_out/gpu_tests.log 2>&1; tail -3 gpurun_out/gpu_tests.log
python tools/tune_jacobi.py 0 > gpurun_out/tune_jacobi.txt 2>&1; cat gpurun_out/tune_jacobi.txt
python tools/tune_gemm.py > gpurun_out/tune_gemm.txt 2>&1; cat gpurun_out/tune_gemm.txt
