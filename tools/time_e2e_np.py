"""End-to-end timing of the cfg2 application through the public API with
numpy in / numpy out (the reference's calling convention); one JSON line.

    python tools/time_e2e_np.py [--reps 5] [--batch 64]
"""
import argparse
import json
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1501_01652_b200 as fh  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--reps", type=int, default=5)
ap.add_argument("--batch", type=int, default=64)
a = ap.parse_args()
n = 2 ** 20
p = fh.select_params(4, n, 1e-15, gamma=4.0)
c = np.random.default_rng(1).standard_normal((a.batch, n)) / np.arange(1, n + 1)
for _ in range(2):
    f = fh.schlomilch_fast(p, c)
ts = []
for _ in range(a.reps):
    torch.cuda.synchronize()
    t = time.perf_counter()
    f = fh.schlomilch_fast(p, c)
    ts.append(time.perf_counter() - t)
t0 = time.perf_counter()
d = np.empty_like(c)
np.copyto(d, c)
tc = time.perf_counter() - t0
print(json.dumps({"ms": 1e3 * float(np.median(ts)), "transforms_per_s": a.batch / float(np.median(ts)),
                  "host_copy_GBs_1thread": c.nbytes / tc / 1e9}))
