"""BASELINE configs[4] scaling sweep on one GPU: Schlomilch nu=0 and the
order-0 DHT for N = 2^lo .. 2^hi at eps in {1e-3, 1e-8, 1e-15}; transforms/s
per cell with CUDA events, plus a sampled-row check against direct fp64 sums
for Schlomilch.  One JSON line per cell.

    python tools/sweep_sizes.py [--task schl|dht] [--lo 10] [--hi 24] [--batch 0]
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
from paper_1501_01652_b200.fourier_bessel import _direct_apply  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--task", default="schl")
ap.add_argument("--lo", type=int, default=10)
ap.add_argument("--hi", type=int, default=24)
ap.add_argument("--eps", default="1e-3,1e-8,1e-15")
ap.add_argument("--budget-gb", type=float, default=8.0, help="coefficient bytes per batch")
a = ap.parse_args()
dev = torch.device("cuda", 0)
for lg in range(a.lo, a.hi + 1):
    n = 2 ** lg
    b = int(max(1, min(256, a.budget_gb * 2 ** 30 / (8 * n * (4 if a.task == "dht" else 1)))))
    rng = np.random.default_rng([lg, 7])
    C = torch.from_numpy(rng.standard_normal((b, n))).to(dev)
    for eps in [float(e) for e in a.eps.split(",")]:
        rec = {"task": a.task, "N": n, "eps": eps, "batch": b}
        try:
            if a.task == "schl":
                p = fh.select_params(0, n, eps)
                fn = lambda: fh.schlomilch_fast(p, C)  # noqa: E731
            else:
                plan = fh.dht_plan(n, eps)
                fn = lambda: fh.dht(plan, C)  # noqa: E731
            F = fn()
            torch.cuda.synchronize()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            reps = 3
            e0.record()
            for _ in range(reps):
                F = fn()
            e1.record()
            torch.cuda.synchronize()
            ms = e0.elapsed_time(e1) / reps
            rec.update(ms=ms, transforms_per_s=b / (ms / 1e3))
            if a.task == "schl":
                rows = np.unique(np.r_[1, 2, n // 3, n // 2, n - 1, n, rng.integers(1, n + 1, 60)])
                k = torch.from_numpy(rows).to(dev)
                out = torch.zeros((1, rows.size), dtype=torch.float64, device=dev)
                col = (torch.arange(1, n + 1, dtype=torch.float64, device=dev) * np.pi).contiguous()
                _direct_apply((k.double() / n).contiguous(), col, n, [0], [dict(vec=0, terms=[(0, 1.0)])],
                              C[:1].contiguous(), out)
                err = float((F[0, k - 1] - out[0]).abs().max())
                tol = 10 * eps * float(C[0].abs().sum())
                rec.update(max_err=err, tol=tol, ok=err <= tol)
        except Exception as exc:  # a cell that cannot run is reported, not fatal
            rec["error"] = repr(exc)[:300]
        print(json.dumps(rec), flush=True)
    del C
    torch.cuda.empty_cache()
