"""One FB (cfg3) or DHT (cfg4) call for ncu captures (plans built and warmed
first; not a benchmark).

    python tools/prof_task.py dht|fb
"""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1501_01652_b200 as fh  # noqa: E402

task = sys.argv[1] if len(sys.argv) > 1 else "dht"
rng = np.random.default_rng(3)
if task == "dht":
    n, b = 2 ** 16, 8
    plan = fh.dht_plan(n, 1e-15)
    C = torch.from_numpy(rng.standard_normal((b, n))).cuda()
    fh.dht(plan, C)
    torch.cuda.synchronize()
    F = fh.dht(plan, C)
else:
    n, b = 2 ** 18, 16
    roots = fh.bessel_roots_j0(n)
    C = torch.from_numpy(rng.uniform(-1, 1, (b, n))).cuda()
    fh.fourier_bessel_eval(0, C, 1e-12, roots=roots)
    torch.cuda.synchronize()
    F = fh.fourier_bessel_eval(0, C, 1e-12, roots=roots)
torch.cuda.synchronize()
print("ok", float(F.abs().sum()))
