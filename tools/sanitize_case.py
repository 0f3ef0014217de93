"""Small invocations of every kernel family, for compute-sanitizer
(memcheck / racecheck / synccheck) runs (tools/sanitize.sh).

    python tools/sanitize_case.py [--big]

Default: cfg2 shape at N=2^14 (four-step pass 1 with TMA stores, pass 2,
narrow-column and narrow-row blocks, reduce), near field, FB (multi-order
near field, direct columns), DHT (chirp-z passes), trig, bessel_j, roots.
--big adds one cfg2 vector at N=2^20 (the bench's exact kernel shapes).
"""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1501_01652_b200 as fh  # noqa: E402

big = "--big" in sys.argv
rng = np.random.default_rng(5)
sizes = [2 ** 14] + ([2 ** 20] if big else [])
for n in sizes:
    c = torch.from_numpy(rng.standard_normal((2, n)) / np.arange(1, n + 1)).cuda()
    f = fh.schlomilch_fast(fh.select_params(4, n, 1e-15, gamma=4.0), c)
    print("schlomilch", n, float(f.abs().sum()))
c = torch.from_numpy(rng.uniform(-1, 1, (2, 4096))).cuda()
print("fb", float(fh.fourier_bessel_eval(0, c, 1e-12).abs().sum()))
plan = fh.dht_plan(2048, 1e-15)
c = torch.from_numpy(rng.standard_normal((2, 2048))).cuda()
print("dht", float(fh.dht(plan, c).abs().sum()))
print("trig", float(np.abs(fh.apply(fh.make_plan(1000, fh.DCT1), rng.standard_normal(1000))).sum()))
print("bessel", float(fh.bessel_j(3, np.linspace(0, 300, 5000)).sum()))
print("direct", float(np.abs(fh.schlomilch_direct(0, 0.0, rng.standard_normal(1024))).sum()))
torch.cuda.synchronize()
print("ok")
