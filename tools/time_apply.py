"""CUDA-event timing of one cfg2-shaped application (far, near or both) for
tuning sweeps; prints one JSON line.  Tunables come from FHTB_* environment
variables (paper_1501_01652_b200/_lib.py).

    python tools/time_apply.py [--flags far] [--batch 64] [--eps 1e-15] [--n 1048576] [--reps 5]
"""
import argparse
import json
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
ap.add_argument("--nu", type=int, default=4)
ap.add_argument("--gamma", type=float, default=4.0)
ap.add_argument("--reps", type=int, default=5)
a = ap.parse_args()
p = fh.select_params(a.nu, a.n, a.eps, gamma=a.gamma)
sc = fh.build_partition(p)
rng = np.random.default_rng(1)
C = torch.from_numpy(rng.standard_normal((a.batch, a.n)) / np.arange(1, a.n + 1)).cuda()
F = torch.zeros_like(C)
g = _grid(p.n, p.gamma, p.m_terms, sc.blocks, sc.mask_segments, [a.nu])
reqs = [dict(vec=v, terms=[(a.nu, 1.0)]) for v in range(a.batch)]
flags = {"far": _lib.FHTB_FAR, "near": _lib.FHTB_NEAR, "both": _lib.FHTB_FAR | _lib.FHTB_NEAR}[a.flags]
for _ in range(2):
    F.zero_()
    g.apply(reqs, C, F, flags)
torch.cuda.synchronize()
ref = F.clone()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
ms = []
for _ in range(a.reps):
    F.zero_()
    e0.record()
    g.apply(reqs, C, F, flags)
    e1.record()
    torch.cuda.synchronize()
    ms.append(e0.elapsed_time(e1))
env = {k: v for k, v in os.environ.items() if k.startswith("FHTB_")}
print(json.dumps({"env": env, "flags": a.flags, "ms": float(np.median(ms)), "ms_all": ms,
                  "checksum": float(ref.abs().sum()), "det": bool(torch.equal(ref, F))}))
