"""bench.py's isolated merge probes alone (merge_range, merge_bitmap dense /
sparse, the binned scatter's fused EAGER push), for A/B of merge kernels.

    python tools/merge_time.py
"""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import bench  # noqa: E402
from paper_2110_14340_b200 import jacc as J  # noqa: E402

out = bench.merge_probes(J)
print(json.dumps({k: {"us": round(v.get("us") or v.get("push_cost_us") or 0, 1),
                      "bytes_pushed": v.get("bytes_pushed")} for k, v in out.items()}), flush=True)
