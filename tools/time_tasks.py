"""The bench.py task timings (FB cfg3, DHT cfg4, cfg2 at looser eps) alone,
one JSON line (for A/B runs with FHTB_LIB)."""
import json
import os
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import bench  # noqa: E402
import paper_1501_01652_b200 as fh  # noqa: E402

torch.cuda.set_device(0)
t = bench.run_tasks(fh, torch.device("cuda", 0), 0, 1, 3, 2)
print(json.dumps({"lib": os.environ.get("FHTB_LIB", "tree"),
                  "tasks": {k: round(v["transforms_per_s"], 2) for k, v in t.items()}}))
