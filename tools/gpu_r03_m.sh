#!/bin/bash
# unfused EAGER merge after the binned scatter: parity + merge probes
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { cat gpurun_out/build.log; exit 1; }
timeout 1500 python -m pytest tests -q -m gpu -x -k "scatter or eager or random_programs or multiprocess or graph" > gpurun_out/tests_m.log 2>&1; tail -2 gpurun_out/tests_m.log
timeout 600 python tools/merge_time.py 2>/dev/null | tail -1
