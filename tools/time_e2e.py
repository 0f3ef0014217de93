"""End-to-end (pinned host in, host out) timing of the cfg2 application
through fhtb_apply_host for several vector-group counts; one JSON line.

    python tools/time_e2e.py [--groups 1,5,8] [--reps 5]
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
from paper_1501_01652_b200.schlomilch import _grid  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--groups", default="1,5,8")
ap.add_argument("--reps", type=int, default=5)
ap.add_argument("--batch", type=int, default=64)
a = ap.parse_args()
n, nu, gamma, eps = 2 ** 20, 4, 4.0, 1e-15
p = fh.select_params(nu, n, eps, gamma=gamma)
sc = fh.build_partition(p)
g = _grid(p.n, p.gamma, p.m_terms, sc.blocks, sc.mask_segments, [nu])
rng = np.random.default_rng(1)
C = torch.from_numpy(rng.standard_normal((a.batch, n)) / np.arange(1, n + 1)).pin_memory()
F = torch.empty_like(C).pin_memory()
reqs = [dict(vec=v, terms=[(nu, 1.0)]) for v in range(a.batch)]
out = {}
for G in [int(x) for x in a.groups.split(",")]:
    for _ in range(2):
        g.apply_host(reqs, C, F, n_groups=G)
    ts = []
    for _ in range(a.reps):
        t0 = time.perf_counter()
        g.apply_host(reqs, C, F, n_groups=G)
        ts.append(time.perf_counter() - t0)
    out[G] = {"ms": 1e3 * float(np.median(ts)), "transforms_per_s": a.batch / float(np.median(ts))}
print(json.dumps(out))
