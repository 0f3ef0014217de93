"""One cfg2-shaped application for ncu captures (not a benchmark: numbers
printed under a profiler are never bench values).

    python tools/prof_apply.py [--flags far|near|both] [--batch 64] [--eps 1e-15] [--reps 1]
"""
import argparse
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1501_01652_b200 as fh  # noqa: E402
from paper_1501_01652_b200 import _lib  # noqa: E402
from paper_1501_01652_b200.schlomilch import _grid  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--flags", default="far")
ap.add_argument("--batch", type=int, default=64)
ap.add_argument("--eps", type=float, default=1e-15)
ap.add_argument("--n", type=int, default=2 ** 20)
ap.add_argument("--reps", type=int, default=1)
a = ap.parse_args()
nu, gamma = 4, 4.0
p = fh.select_params(nu, a.n, a.eps, gamma=gamma)
sc = fh.build_partition(p)
rng = np.random.default_rng(1)
C = torch.from_numpy(rng.standard_normal((a.batch, a.n)) / np.arange(1, a.n + 1)).cuda()
F = torch.zeros_like(C)
g = _grid(p.n, p.gamma, p.m_terms, sc.blocks, sc.mask_segments, [nu])
reqs = [dict(vec=v, terms=[(nu, 1.0)]) for v in range(a.batch)]
flags = {"far": _lib.FHTB_FAR, "near": _lib.FHTB_NEAR, "both": _lib.FHTB_FAR | _lib.FHTB_NEAR}[a.flags]
for _ in range(a.reps):
    g.apply(reqs, C, F, flags)
torch.cuda.synchronize()
print("ok", float(F.abs().sum()))
