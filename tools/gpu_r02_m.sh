#!/bin/bash
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || exit 1
for r in 1 2; do timeout 300 python tools/time_loop.py himeno_copy 10; timeout 300 python tools/time_loop.py himeno 5; done
timeout 900 python -m pytest tests/test_gpu_parity.py -q -m gpu -x -k "himeno or gemm" 2>&1 | tail -2
