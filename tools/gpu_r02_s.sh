#!/bin/bash
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { cat gpurun_out/build.log; exit 1; }
timeout 1500 python -m pytest tests/test_gpu_parity.py tests/test_gpu_random_programs.py tests/test_gpu_multiprocess.py -q -m gpu --timeout 900 -k "scatter or graph or random or fig4 or multiprocess or mp" > gpurun_out/gpu_tests_s.log 2>&1
tail -3 gpurun_out/gpu_tests_s.log
bash tools/gpu_sanitize.sh
python - <<'PY'
import sys, json
sys.path.insert(0, ".")
import bench
from paper_2110_14340_b200 import jacc as J
m = bench.merge_probes(J)
print(json.dumps(m["binned_scatter_fused_push"]))
print(json.dumps(m["merge_bitmap_dense"]))
PY
for l in scat_f64 scat_i32; do timeout 300 python tools/time_loop.py $l 8; done
