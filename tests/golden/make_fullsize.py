"""Generate FULL-SIZE reference fixtures (sampled rows) by running the
REFERENCE package in the build container.

    PYTHONDONTWRITEBYTECODE=1 python tests/golden/make_fullsize.py [-j 8] [--only NAME,...]

The BASELINE.json configurations are too large to store whole, so each case
stores only:
  * how to regenerate its inputs (numpy PCG64 seed words; numpy's PCG64
    stream is stable, so the GPU box draws the same bits),
  * a set of sampled output rows spanning every partition block (first/last
    rows, the partition edges a_p, b_p and their neighbours, random rows),
  * the reference's FAST output at those rows where the reference finishes
    in minutes (`schlomilch_fast`, `fourier_bessel_eval`, `dht`), and
  * a DIRECT fp64 sum at those rows computed with the reference's own
    `bessel_j` (and `_rows_direct` for the DHT), i.e. independent of the
    CUDA Bessel evaluator the GPU near field and direct kernels share.
Trig cases store sampled outputs plus a checksum (w . out) with a seeded w.
Bessel cases pin J_nu at large arguments (to 4e6) in every dispatch range.

Writes tests/golden/fullsize.npz and tests/golden/fullsize.json.  Each case
is computed in its own worker process and cached under /tmp/fullsize_cache,
so an interrupted run resumes.
"""

import argparse
import importlib
import json
import math
import os
import pickle
import sys
import time
from concurrent.futures import ProcessPoolExecutor

import numpy as np

REF = "/root/reference/pkg/src"
HERE = os.path.dirname(os.path.abspath(__file__))
CACHE = "/tmp/fullsize_cache"
SEED = 1501          # bench.py SEED: cfg2 vectors are rng([SEED, N, b])
TASK_SEED = 1508     # bench.py task vectors: rng([SEED + 7, N, b])


def _ref():
    sys.dont_write_bytecode = True
    if REF not in sys.path:
        sys.path.insert(0, REF)
    import fasthankel as fh
    return fh


# --------------------------------------------------------------------------
# inputs (mirrored by tests/test_gpu_fullsize_ref.py)

def cfg2_vector(n, b=0):
    g = np.random.default_rng([SEED, n, b]).standard_normal(n)
    return g / np.arange(1, n + 1, dtype=float)


def task_vector(kind, n, b=0):
    g = np.random.default_rng([TASK_SEED, n, b])
    return g.uniform(-1.0, 1.0, n) if kind == "u" else g.standard_normal(n)


def sweep_vector(n):
    return np.random.default_rng([SEED, n, 9]).standard_normal(n)


def sample_rows(n, count, seed, edges=()):
    rng = np.random.default_rng([seed, n])
    rows = set(rng.integers(1, n + 1, count).tolist())
    rows |= {1, 2, 3, 4, n - 1, n} | {max(1, int(n * f)) for f in (0.001, 0.01, 0.1, 0.5, 0.9)}
    for e in edges:
        rows |= {e - 1, e, e + 1}
    return np.array(sorted(r for r in rows if 1 <= r <= n), dtype=np.int64)


def schl_edges(fh, nu, n, eps, gamma):
    p = fh.select_params(nu, n, eps, gamma=gamma)
    sc = fh.build_partition(p)
    e = set()
    for (r0, r1), (c0, c1) in sc.blocks:
        e |= {r0, r1}
    return sorted(x for x in e if 1 <= x <= n)


# --------------------------------------------------------------------------
# direct sums with the reference bessel_j

def direct_rows_schl(fh, nu, gamma, c, rows, chunk=8):
    n = c.shape[0]
    omega = (np.arange(1, n + 1, dtype=float) + gamma) * math.pi
    out = np.empty(rows.size)
    for i in range(0, rows.size, chunk):
        r = rows[i:i + chunk].astype(float) / n
        z = np.multiply.outer(r, omega)
        out[i:i + chunk] = fh.bessel_j(nu, z) @ c
    return out


def newton_roots(fh, count):
    """j_{0,n}, n = 1..count, by the reference's Newton iteration
    (bessel.py:295-321) with the reference's bessel_j, WITHOUT its 1e-13
    residual gate (fp64 cannot meet it beyond ~2e6)."""
    n = np.arange(1, count + 1, dtype=float)
    z = (n - 0.25) * math.pi
    for _ in range(20):
        step = fh.bessel_j(0, z) / fh.bessel_j(1, z)
        z = z + step
        if np.max(np.abs(step)) <= 4.0 * 2.0 ** -52 * z[-1]:
            break
    return z


def direct_rows_dht(fh, roots, c, rows, chunk=8):
    n = c.shape[0]
    out = np.empty(rows.size)
    for i in range(0, rows.size, chunk):
        scale = roots[rows[i:i + chunk] - 1] / roots[n]
        z = np.multiply.outer(scale, roots[:n])
        out[i:i + chunk] = fh.bessel_j(0, z) @ c
    return out


# --------------------------------------------------------------------------
# cases: name -> function returning (meta dict, arrays dict)

def case_cfg2(eps):
    def run():
        fh = _ref()
        n, nu, gamma = 2 ** 20, 4, 4.0
        c = cfg2_vector(n, 0)
        rows = sample_rows(n, 200, 11, schl_edges(fh, nu, n, 1e-15, gamma) + schl_edges(fh, nu, n, eps, gamma))
        t = time.time()
        f = fh.schlomilch_fast(fh.select_params(nu, n, eps, gamma=gamma), c)
        meta = dict(task="schlomilch", n=n, nu=nu, gamma=gamma, eps=eps, input="cfg2", b=0,
                    ref_fast_seconds=time.time() - t, l1=float(np.abs(c).sum()))
        return meta, {"rows": rows, "fast": f[rows - 1]}
    return run


def case_cfg2_direct():
    fh = _ref()
    n, nu, gamma = 2 ** 20, 4, 4.0
    c = cfg2_vector(n, 0)
    rows = sample_rows(n, 200, 11, sorted(set(sum((schl_edges(fh, nu, n, e, gamma) for e in (1e-3, 1e-8, 1e-15)), []))))
    t = time.time()
    d = direct_rows_schl(fh, nu, gamma, c, rows)
    meta = dict(task="schlomilch_direct", n=n, nu=nu, gamma=gamma, input="cfg2", b=0,
                ref_direct_seconds=time.time() - t, l1=float(np.abs(c).sum()))
    return meta, {"rows": rows, "direct": d}


def case_fb_cfg3():
    fh = _ref()
    n, eps = 2 ** 18, 1e-12
    c = task_vector("u", n, 0)
    roots = fh.bessel_roots_j0(n)
    rows = sample_rows(n, 200, 5, [19, 20, 21, 64, 512, 4096])
    t = time.time()
    f = fh.fourier_bessel_eval(0, c, eps, roots=roots)
    tf = time.time() - t
    r = np.asarray(roots.roots)
    d = np.empty(rows.size)
    for i in range(0, rows.size, 8):
        z = np.multiply.outer(rows[i:i + 8].astype(float) / n, r)
        d[i:i + 8] = fh.bessel_j(0, z) @ c
    meta = dict(task="fb", n=n, nu=0, eps=eps, input="task_u", b=0, ref_fast_seconds=tf,
                l1=float(np.abs(c).sum()))
    return meta, {"rows": rows, "fast": f[rows - 1], "direct": d}


def case_dht_cfg4_direct():
    fh = _ref()
    dhtmod = importlib.import_module("fasthankel.dht")
    n, eps = 2 ** 16, 1e-15
    c = task_vector("n", n, 0)
    plan = fh.dht_plan(n, eps)
    rows = sample_rows(n, 200, 6, list(range(1, 30)))
    d = np.empty(rows.size)
    for i, k in enumerate(rows):
        d[i] = dhtmod._rows_direct(plan, c, int(k), int(k) + 1)[0]
    meta = dict(task="dht_direct", n=n, eps=eps, input="task_n", b=0, l1=float(np.abs(c).sum()))
    return meta, {"rows": rows, "direct": d}


def case_dht_cfg4_fast():
    fh = _ref()
    n, eps = 2 ** 16, 1e-15
    c = task_vector("n", n, 0)
    plan = fh.dht_plan(n, eps)
    rows = sample_rows(n, 200, 6, list(range(1, 30)))
    t = time.time()
    st = {}
    f = fh.dht(plan, c, stats=st)
    meta = dict(task="dht", n=n, eps=eps, input="task_n", b=0, ref_fast_seconds=time.time() - t,
                l1=float(np.abs(c).sum()), stats=st)
    # the whole output vector is only 512 KiB: keep it all
    return meta, {"rows": rows, "fast": f[rows - 1], "full": f}


def case_dht_fast(n, eps):
    def run():
        fh = _ref()
        c = sweep_vector(n)
        plan = fh.dht_plan(n, eps)
        rows = sample_rows(n, 128, 7, list(range(1, 30)))
        t = time.time()
        f = fh.dht(plan, c)
        meta = dict(task="dht", n=n, eps=eps, input="sweep", ref_fast_seconds=time.time() - t,
                    l1=float(np.abs(c).sum()))
        return meta, {"rows": rows, "fast": f[rows - 1], "full": f}
    return run


def case_schl_sweep_fast(n, eps):
    def run():
        fh = _ref()
        c = sweep_vector(n)
        rows = sample_rows(n, 200, 12, schl_edges(fh, 0, n, eps, 0.0))
        t = time.time()
        f = fh.schlomilch_fast(fh.select_params(0, n, eps), c)
        meta = dict(task="schlomilch", n=n, nu=0, gamma=0.0, eps=eps, input="sweep",
                    ref_fast_seconds=time.time() - t, l1=float(np.abs(c).sum()))
        return meta, {"rows": rows, "fast": f[rows - 1]}
    return run


def case_schl_sweep_direct(n, count):
    def run():
        fh = _ref()
        c = sweep_vector(n)
        edges = sorted(set(sum((schl_edges(fh, 0, n, e, 0.0) for e in (1e-3, 1e-8, 1e-15)), [])))
        rows = sample_rows(n, count, 13, edges)
        t = time.time()
        d = direct_rows_schl(fh, 0, 0.0, c, rows, chunk=2 if n > 2 ** 21 else 8)
        meta = dict(task="schlomilch_direct", n=n, nu=0, gamma=0.0, input="sweep",
                    ref_direct_seconds=time.time() - t, l1=float(np.abs(c).sum()))
        return meta, {"rows": rows, "direct": d}
    return run


def case_dht_sweep_direct(n, count):
    def run():
        fh = _ref()
        c = sweep_vector(n)
        roots = newton_roots(fh, n + 1)
        rows = sample_rows(n, count, 14, list(range(1, 30)))
        t = time.time()
        d = direct_rows_dht(fh, roots, c, rows, chunk=2 if n > 2 ** 21 else 8)
        meta = dict(task="dht_direct", n=n, input="sweep", ref_direct_seconds=time.time() - t,
                    l1=float(np.abs(c).sum()))
        return meta, {"rows": rows, "direct": d}
    return run


def case_bessel_large():
    fh = _ref()
    from fasthankel.bessel import _dispatch_cutoffs
    meta = dict(task="bessel", orders=[])
    arrays = {}
    rng = np.random.default_rng(77)
    for nu in (0, 1, 2, 3, 4, 5, 8, 10, 11, 16, 20, 32, 40, 63):
        t_lo, s_hi = _dispatch_cutoffs(nu)
        z = np.concatenate([np.logspace(-3, math.log10(4.2e6), 1500),
                            np.linspace(0.0, 2.5 * s_hi, 1200),
                            s_hi * (1 + np.linspace(-1e-3, 1e-3, 41)),
                            t_lo * (1 + np.linspace(-1e-3, 1e-3, 41)),
                            rng.uniform(1e4, 4.2e6, 500)])
        arrays["z_%d" % nu] = z
        arrays["j_%d" % nu] = fh.bessel_j(nu, z)
        meta["orders"].append(dict(nu=nu, t_lo=t_lo, s_hi=s_hi))
    return meta, arrays


def case_bessel_mp():
    """J_nu to 30 digits (mpmath) at large arguments: the reference's own
    Hankel path rounds its phase z - (2 nu + 1) pi / 4 to fp64, which is off
    by up to ulp(z)/2 rad (1.5e-13 absolute at z = 4.2e6), so the large-z
    check uses these values (the reference's values pin it below ~1e4)."""
    import mpmath as mp
    _ref()
    from fasthankel.bessel import _dispatch_cutoffs
    mp.mp.dps = 30
    meta = dict(task="bessel_mp", orders=[])
    arrays = {}
    rng = np.random.default_rng(91)
    for nu in (0, 1, 4, 10, 40, 63):
        t_lo, s_hi = _dispatch_cutoffs(nu)
        z = np.concatenate([np.logspace(1, math.log10(4.2e6), 60), rng.uniform(1e5, 4.2e6, 40),
                            s_hi * (1 + np.linspace(-1e-3, 1e-3, 5)), np.linspace(0.5, 2.5 * s_hi, 20)])
        arrays["z_%d" % nu] = z
        arrays["j_%d" % nu] = np.array([float(mp.besselj(nu, mp.mpf(float(x)))) for x in z])
        meta["orders"].append(nu)
    return meta, arrays


def case_trig():
    fh = _ref()
    meta = dict(task="trig", cases=[])
    arrays = {}
    for n in (4095, 4096, 4097, 8191, 8193, 65536, 65537, 2 ** 20 - 1, 2 ** 20 + 1):
        for kind in (fh.DCT1, fh.DST1):
            b = 2 if n < 100000 else 1
            v = np.random.default_rng([77, n, kind == fh.DST1]).standard_normal((b, n))
            w = np.random.default_rng([78, n]).standard_normal(n)
            out = fh.apply(fh.make_plan(n, kind), v)
            idx = np.unique(np.concatenate([np.arange(4), n - 4 + np.arange(4),
                                            np.random.default_rng([79, n]).integers(0, n, 256)]))
            key = "%s_%d" % (kind, n)
            arrays[key + "_idx"] = idx
            arrays[key + "_val"] = out[:, idx]
            arrays[key + "_chk"] = out @ w
            arrays[key + "_l1"] = np.abs(v).sum(1)
            meta["cases"].append(dict(kind=kind, n=n, batch=b))
    return meta, arrays


def case_high_order():
    """Orders beyond the round-1 engine caps (nu > 63; FB universes > 16)."""
    fh = _ref()
    meta = dict(task="high_order", cases=[])
    arrays = {}
    for (nu, n, eps) in ((64, 4096, 1e-8), (80, 4096, 1e-8), (100, 2048, 1e-15), (70, 1000, 1e-3)):
        c = np.random.default_rng([80, nu, n]).standard_normal(n)
        f = fh.schlomilch_fast(fh.select_params(nu, n, eps), c)
        key = "schl_%d_%d" % (nu, n)
        arrays[key] = f
        meta["cases"].append(dict(kind="schlomilch", nu=nu, n=n, eps=eps, gamma=0.0, key=key))
    for (nu, n, eps) in ((60, 2048, 1e-15), (20, 1024, 1e-15)):
        c = np.random.default_rng([81, nu, n]).uniform(-1, 1, n)
        f = fh.fourier_bessel_eval(nu, c, eps)
        key = "fb_%d_%d" % (nu, n)
        arrays[key] = f
        meta["cases"].append(dict(kind="fb", nu=nu, n=n, eps=eps, key=key))
    for nu in (64, 80, 100, 150):
        z = np.concatenate([np.linspace(0, 600, 1201), np.logspace(-2, 6, 400)])
        arrays["bj_z_%d" % nu] = z
        arrays["bj_%d" % nu] = fh.bessel_j(nu, z)
        meta["cases"].append(dict(kind="bessel", nu=nu, key="bj_%d" % nu))
    return meta, arrays


CASES = {
    "cfg2_eps1e-3": case_cfg2(1e-3),
    "cfg2_eps1e-8": case_cfg2(1e-8),
    "cfg2_eps1e-15": case_cfg2(1e-15),
    "cfg2_direct": case_cfg2_direct,
    "fb_cfg3": case_fb_cfg3,
    "dht_cfg4_direct": case_dht_cfg4_direct,
    "dht_cfg4_fast": case_dht_cfg4_fast,
    "dht_4096_eps1e-15": case_dht_fast(4096, 1e-15),
    "dht_16384_eps1e-8": case_dht_fast(16384, 1e-8),
    "schl_2^18_eps1e-3": case_schl_sweep_fast(2 ** 18, 1e-3),
    "schl_2^18_eps1e-8": case_schl_sweep_fast(2 ** 18, 1e-8),
    "schl_2^18_eps1e-15": case_schl_sweep_fast(2 ** 18, 1e-15),
    "schl_2^20_eps1e-15": case_schl_sweep_fast(2 ** 20, 1e-15),
    "schl_2^18_direct": case_schl_sweep_direct(2 ** 18, 160),
    "schl_2^20_direct": case_schl_sweep_direct(2 ** 20, 120),
    "schl_2^22_direct": case_schl_sweep_direct(2 ** 22, 48),
    "schl_2^24_direct": case_schl_sweep_direct(2 ** 24, 24),
    "dht_2^18_direct": case_dht_sweep_direct(2 ** 18, 96),
    "dht_2^20_direct": case_dht_sweep_direct(2 ** 20, 64),
    "dht_2^22_direct": case_dht_sweep_direct(2 ** 22, 40),
    "dht_2^24_direct": case_dht_sweep_direct(2 ** 24, 24),
    "bessel_large": case_bessel_large,
    "bessel_mp": case_bessel_mp,
    "trig": case_trig,
    "high_order": case_high_order,
}


def _run(name):
    path = os.path.join(CACHE, name + ".pkl")
    if os.path.exists(path):
        return name, "cached"
    os.environ["OPENBLAS_NUM_THREADS"] = "1"
    t = time.time()
    meta, arrays = CASES[name]()
    meta["gen_seconds"] = time.time() - t
    with open(path + ".tmp", "wb") as f:
        pickle.dump((meta, arrays), f)
    os.replace(path + ".tmp", path)
    return name, "%.0fs" % (time.time() - t)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("-j", type=int, default=os.cpu_count() or 1)
    ap.add_argument("--only", default="")
    ap.add_argument("--collect-only", action="store_true")
    ap.add_argument("--merge", action="store_true",
                    help="keep the cases already in fullsize.npz/json and add or replace the cached ones")
    a = ap.parse_args()
    os.makedirs(CACHE, exist_ok=True)
    names = [x for x in a.only.split(",") if x] or list(CASES)
    # longest first
    slow = ["dht_cfg4_fast", "dht_2^24_direct", "schl_2^24_direct", "dht_16384_eps1e-8", "cfg2_eps1e-15"]
    names = sorted(names, key=lambda x: (x not in slow, slow.index(x) if x in slow else 0))
    if not a.collect_only:
        with ProcessPoolExecutor(a.j) as ex:
            for name, how in ex.map(_run, names):
                print(name, how, flush=True)
    meta, arrays = {}, {}
    if a.merge:
        with open(os.path.join(HERE, "fullsize.json")) as f:
            meta = json.load(f)
        with np.load(os.path.join(HERE, "fullsize.npz")) as old:
            arrays = {k: old[k] for k in old.files}
    for name in CASES:
        p = os.path.join(CACHE, name + ".pkl")
        if not os.path.exists(p):
            if name not in meta:
                print("missing", name)
            continue
        with open(p, "rb") as f:
            m, arr = pickle.load(f)
        meta[name] = m
        for k, v in arr.items():
            arrays[name + "/" + k] = v
    np.savez_compressed(os.path.join(HERE, "fullsize.npz"), **arrays)
    with open(os.path.join(HERE, "fullsize.json"), "w") as f:
        json.dump(meta, f, indent=1, sort_keys=True)
    print("wrote", len(meta), "cases,", len(arrays), "arrays")


if __name__ == "__main__":
    main()
