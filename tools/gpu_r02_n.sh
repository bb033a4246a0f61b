#!/bin/bash
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || exit 1
python - <<'PY'
import sys, json
sys.path.insert(0, ".")
import bench
from paper_2110_14340_b200 import jacc as J
for r in range(2):
    print(json.dumps(bench.merge_probes(J)))
PY
