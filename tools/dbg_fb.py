import sys, os, time, cProfile, pstats
sys.path.insert(0, os.getcwd())
import numpy as np, torch
import paper_1501_01652_b200 as fh
n, B = 2 ** 20, 16
roots = fh.bessel_roots_j0(n)
C = torch.from_numpy(np.random.default_rng(1).uniform(-1, 1, (B, n))).cuda()
for _ in range(2):
    fh.fourier_bessel_eval(0, C, 1e-12, roots=roots)
torch.cuda.synchronize()
t = time.perf_counter()
for _ in range(3):
    fh.fourier_bessel_eval(0, C, 1e-12, roots=roots)
torch.cuda.synchronize()
print("ms per call", (time.perf_counter() - t) / 3 * 1e3)
pr = cProfile.Profile()
pr.enable()
fh.fourier_bessel_eval(0, C, 1e-12, roots=roots)
torch.cuda.synchronize()
pr.disable()
pstats.Stats(pr).sort_stats("cumulative").print_stats(18)
