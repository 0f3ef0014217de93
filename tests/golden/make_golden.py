"""Generate golden input/output vectors by running the REFERENCE package.

Run in the build container only (the reference lives at /root/reference and
does not exist on the GPU box):

    PYTHONDONTWRITEBYTECODE=1 python tests/golden/make_golden.py

Writes tests/golden/golden.npz (arrays) and tests/golden/golden.json
(planner outputs, stats counters, case index).  The fixtures pin both the
CPU oracle (oracle/fht_oracle.py) and the CUDA path.
"""

import importlib
import json
import math
import os
import sys

import numpy as np

REF = "/root/reference/pkg/src"
HERE = os.path.dirname(os.path.abspath(__file__))


def main():
    sys.dont_write_bytecode = True
    sys.path.insert(0, REF)
    import fasthankel as fh
    dhtmod = importlib.import_module("fasthankel.dht")  # fasthankel.dht is the function
    from fasthankel.schlomilch import _select_params, SchlomilchEngine

    arrays = {}
    meta = {"bessel": [], "trig": [], "params": [], "schlomilch": [], "block": [],
            "engine": [], "fb": [], "dht": [], "roots": None, "neumann": [],
            "selfinv": []}

    # ---- Bessel point values -------------------------------------------
    rng = np.random.default_rng(2024)
    zgrid = np.concatenate([np.linspace(0.0, 200.0, 801), rng.uniform(0, 120, 400),
                            [1e-8, 1e-3, 0.165, 2.404825557695773, 17.8, 30.8]])
    arrays["bessel_z"] = zgrid
    for nu in (0, 1, 2, 3, 4, 5, 7, 10, 15, 20):
        arrays["bessel_j_%d" % nu] = fh.bessel_j(nu, zgrid)
        meta["bessel"].append(nu)
    zh = np.linspace(17.8, 80.0, 200)
    arrays["hankel_z"] = zh
    arrays["hankel_0_10"] = fh.hankel_asy_eval(0, 10, zh)
    arrays["hankel_3_6"] = fh.hankel_asy_eval(3, 6, zh)
    zt = np.linspace(0.0, 1.4, 100)
    arrays["taylor_z"] = zt
    arrays["taylor_0_5"] = fh.taylor_eval(0, 5, zt)
    arrays["taylor_2_9"] = fh.taylor_eval(2, 9, zt)

    # ---- roots ------------------------------------------------------------
    tab = fh.bessel_roots_j0(3001)
    arrays["roots"] = np.array(tab.roots)
    arrays["perturb"] = np.array(tab.perturbations)
    arrays["ratio_500"] = tab.ratio_perturbation(np.arange(1, 501), 500)
    meta["roots"] = 3001

    # ---- trig -------------------------------------------------------------
    for n in (1, 2, 3, 5, 9, 16, 17, 33, 64, 65, 100, 500, 1023, 1024, 1025):
        for kind in (fh.DCT1, fh.DST1):
            if kind == fh.DCT1 and n < 2:
                continue
            v = np.random.default_rng(n * 7 + (kind == fh.DST1)).standard_normal((3, n))
            key = "trig_%s_%d" % (kind, n)
            arrays[key + "_in"] = v
            arrays[key + "_out"] = fh.apply(fh.make_plan(n, kind), v)
            meta["trig"].append([kind, n])
    vc = np.random.default_rng(44).standard_normal(33) + 1j * np.random.default_rng(45).standard_normal(33)
    arrays["trig_cplx_in"] = vc
    arrays["trig_cplx_dct"] = fh.apply(fh.make_plan(33, fh.DCT1), vc)
    arrays["trig_cplx_dst"] = fh.apply(fh.make_plan(33, fh.DST1), vc)

    # ---- planner ------------------------------------------------------------
    for nu in (0, 1, 2, 4, 10):
        for n in (1, 2, 10, 20, 21, 158, 159, 500, 4096, 65536, 2 ** 18, 2 ** 20, 2 ** 24, 100000):
            for eps in (1e-3, 1e-8, 1e-12, 1e-15, 1e-17):
                for gamma in (0.0, -0.25, 4.0):
                    p = _select_params(nu, n, eps, gamma)
                    sc = fh.build_partition(p)
                    meta["params"].append(dict(
                        nu=nu, n=n, eps=eps, gamma=gamma, m=p.m_terms, s=p.s,
                        alpha=p.alpha, beta=p.beta, P=p.partitions,
                        blocks=[list(map(list, b)) for b in sc.blocks],
                        segments=[list(s) for s in sc.mask_segments],
                        row_min=sc.row_min, mask=sc.mask_size()))
    for eps in (1e-3, 1e-8, 1e-12, 1e-15):
        for margin in (1.0, 1.01):
            q = fh.select_neumann_params(eps, margin)
            meta["neumann"].append(dict(eps=eps, margin=margin, K=q.k_terms, T=q.t_terms,
                                        p=q.p_cut, q=q.q_cut, n_split=q.n_split))

    # ---- Schlomilch evaluations -----------------------------------------------
    cases = [
        # (n, nu, gamma, eps, kind, seed)
        (10, 10, 0.0, 1e-3, "normal", 4),
        (64, 0, 0.0, 1e-8, "normal", 0),
        (100, 0, 0.0, 1e-15, "normal", 100),
        (158, 0, 0.0, 1e-15, "normal", 158),
        (200, 0, 0.0, 1e-15, "normal", 17),
        (300, 0, 0.0, 1e-13, "complex", 3),
        (400, 0, -0.25, 1e-15, "normal", 10),
        (500, 2, 0.0, 1e-8, "normal", 502),
        (500, 2, 0.5, 1e-8, "normal", 9),
        (700, 0, 0.0, 1e-8, "normal", 12),
        (1024, 1, 0.0, 1e-3, "normal", 31),
        (1024, 10, 0.0, 1e-15, "normal", 32),
        (2000, 0, 0.0, 1e-15, "normal", 2000),
        (2048, 4, 4.0, 1e-15, "cfg2", 7),
        (4096, 0, 0.0, 1e-15, "normal", 4096),
        (4096, 4, 4.0, 1e-8, "cfg2", 8),
        (4096, 4, 4.0, 1e-3, "cfg2", 9),
    ]
    for i, (n, nu, gamma, eps, kind, seed) in enumerate(cases):
        g = np.random.default_rng(seed)
        if kind == "complex":
            c = g.standard_normal(n) + 1j * g.standard_normal(n)
        elif kind == "cfg2":
            c = g.standard_normal(n) / np.arange(1, n + 1)
        else:
            c = g.standard_normal(n)
        p = fh.select_params(nu, n, eps, gamma=gamma)
        st = {}
        arrays["schl_%d_c" % i] = c
        arrays["schl_%d_fast" % i] = fh.schlomilch_fast(p, c, stats=st)
        arrays["schl_%d_single" % i] = fh.schlomilch_single_partition(p, c)
        if n <= 2048:
            arrays["schl_%d_direct" % i] = fh.schlomilch_direct(nu, gamma, c)
        meta["schlomilch"].append(dict(i=i, n=n, nu=nu, gamma=gamma, eps=eps, kind=kind,
                                       stats=st, has_direct=n <= 2048))

    # ---- single asymptotic blocks ---------------------------------------------
    for i, (n, nu, eps, rows, cols, seed) in enumerate([
            (64, 0, 1e-8, None, None, 0), (64, 1, 1e-8, (40, 60), (30, 65), 5),
            (1024, 3, 1e-15, (300, 1025), (200, 900), 6)]):
        p = fh.select_params(nu, n, eps)
        lo = math.ceil(p.alpha * math.sqrt(n))
        rows = rows or (lo, n + 1)
        cols = cols or (lo, n + 1)
        c = np.random.default_rng(seed).standard_normal(n)
        st = {}
        arrays["block_%d_c" % i] = c
        arrays["block_%d_out" % i] = fh.asy_block_apply(p, rows, cols, c, st)
        meta["block"].append(dict(i=i, n=n, nu=nu, eps=eps, rows=list(rows), cols=list(cols),
                                  stats=st))

    # ---- multi-order engine -------------------------------------------------------
    for i, (n, gamma, eps, orders) in enumerate([(512, -0.25, 1e-12, [0, 1, 2, 3]),
                                                  (1000, 0.0, 1e-15, [0, 2, 5])]):
        eng = SchlomilchEngine(n, gamma, eps, orders)
        g = np.random.default_rng(77 + i)
        reqs = [(((orders[0], 1.0),), g.standard_normal(n)),
                (((orders[1], 0.5), (orders[-1], -0.25)), g.standard_normal(n)),
                (tuple((o, 0.1 * (j + 1)) for j, o in enumerate(orders)), g.uniform(-1, 1, n))]
        st = {}
        ys = eng.apply_many(reqs, st)
        for j, (ow, c) in enumerate(reqs):
            arrays["eng_%d_%d_c" % (i, j)] = c
            arrays["eng_%d_%d_y" % (i, j)] = ys[j]
        meta["engine"].append(dict(i=i, n=n, gamma=gamma, eps=eps, orders=orders,
                                   reqs=[[list(map(list, ow))] for ow, _ in reqs], stats=st,
                                   m=eng.params.m_terms, s=eng.params.s, P=eng.params.partitions))

    # ---- Fourier-Bessel -----------------------------------------------------------
    fb_cases = [(64, 0, 1e-15, "normal"), (256, 0, 1e-3, "normal"), (256, 1, 1e-8, "normal"),
                (1024, 0, 1e-15, "normal"), (1024, 1, 1e-15, "normal"), (1024, 0, 1e-8, "normal"),
                (2048, 0, 1e-12, "uniform"), (10, 0, 1e-15, "normal"), (500, 1, 1e-8, "normal")]
    for i, (n, nu, eps, kind) in enumerate(fb_cases):
        g = np.random.default_rng(900 + i)
        c = g.uniform(-1, 1, n) if kind == "uniform" else g.standard_normal(n)
        st = {}
        arrays["fb_%d_c" % i] = c
        arrays["fb_%d_fast" % i] = fh.fourier_bessel_eval(nu, c, eps, stats=st)
        st2 = {}
        arrays["fb_%d_prune" % i] = fh.fourier_bessel_eval(nu, c, eps, stats=st2, prune=True)
        arrays["fb_%d_direct" % i] = fh.fourier_bessel_direct(nu, c)
        meta["fb"].append(dict(i=i, n=n, nu=nu, eps=eps, kind=kind, stats=st, stats_prune=st2))

    # ---- DHT -------------------------------------------------------------------------
    dht_cases = [(1, 1e-15), (10, 1e-8), (23, 1e-15), (64, 1e-3), (64, 1e-15), (256, 1e-8),
                 (256, 1e-15), (1024, 1e-3), (1024, 1e-15), (2048, 1e-15)]
    for i, (n, eps) in enumerate(dht_cases):
        plan = dhtmod.dht_plan(n, eps)
        c = np.random.default_rng(500 + i).standard_normal(n)
        st = {}
        arrays["dht_%d_c" % i] = c
        arrays["dht_%d_fast" % i] = dhtmod.dht(plan, c, stats=st)
        arrays["dht_%d_direct" % i] = dhtmod.dht_direct(plan, c)
        arrays["dht_%d_weights" % i] = plan.weights
        meta["dht"].append(dict(i=i, n=n, eps=eps, stats=st, K=plan.k_terms, T=plan.t_terms,
                                row_split=plan.row_split))
    for i, (n, eps) in enumerate([(128, 1e-15), (512, 1e-15)]):
        c = np.random.default_rng(600 + i).standard_normal(n)
        arrays["selfinv_%d_c" % i] = c
        r = dhtmod.dht_self_inverse_residual(n, eps, c)
        meta["selfinv"].append(dict(i=i, n=n, eps=eps, residual=r))

    np.savez_compressed(os.path.join(HERE, "golden.npz"), **arrays)
    with open(os.path.join(HERE, "golden.json"), "w") as f:
        json.dump(meta, f, indent=0, sort_keys=True)
    print("wrote", len(arrays), "arrays")


if __name__ == "__main__":
    main()
