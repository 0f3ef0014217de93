import sys, os, time, cProfile, pstats
sys.path.insert(0, os.getcwd())
import numpy as np, torch
import paper_1501_01652_b200 as fh
n, B = 2 ** 16, 8
plan = fh.dht_plan(n, 1e-15)
C = torch.from_numpy(np.random.default_rng(1).standard_normal((B, n))).cuda()
for _ in range(2):
    fh.dht(plan, C)
torch.cuda.synchronize()
for rep in range(2):
    t = time.perf_counter()
    for _ in range(3):
        fh.dht(plan, C)
    torch.cuda.synchronize()
    print("ms per call", (time.perf_counter() - t) / 3 * 1e3)
pr = cProfile.Profile()
pr.enable()
t = time.perf_counter()
fh.dht(plan, C)
t1 = time.perf_counter()
torch.cuda.synchronize()
pr.disable()
print("host ms", (t1 - t) * 1e3, "total", (time.perf_counter() - t) * 1e3)
pstats.Stats(pr).sort_stats("tottime").print_stats(12)
