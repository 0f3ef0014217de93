"""Benchmark: transforms/s of the fast Schlomilch/FB/DHT hot path on B200.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]

Headline workload (BASELINE.json configs[1], "cfg2"): Schlomilch expansion
nu=4, omega_n=(n+4)pi, r_k=k/N, N=2^20, 64 vectors c_n = g_n/n, g ~ N(0,1)
(seeded), eps=1e-15, fp64.  One step = one application of the partitioned
scheme (fused DCT-I/DST-I far field + DMMA near field) to the 64 vectors,
inputs resident in HBM (512 MiB, larger than the 126 MB L2, so no flush is
needed between steps).  Under torchrun every rank runs its own 64 vectors
(weak scaling, no data-path collective); value = all vectors / max-rank time.

--impl reference runs the CPU oracle (oracle/fht_oracle.py, a NumPy port of
the reference, which cannot travel to the GPU box) on the same config.
"""

import argparse
import json
import math
import os
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "transforms/s at N=2^20 fp64 (Schlomilch cfg2: nu=4, gamma=4, eps=1e-15, 64 vectors)"
UNIT = "transforms/s"
N_DEF, NU, GAMMA, EPS, BATCH = 2 ** 20, 4, 4.0, 1e-15, 64
SEED = 1501


def make_inputs(n, batch, rank):
    rows = []
    idx = np.arange(1, n + 1, dtype=float)
    for b in range(batch):
        g = np.random.default_rng([SEED, n, rank * batch + b]).standard_normal(n)
        rows.append(g / idx)
    return np.stack(rows)


def model_bytes(params, scheme):
    """bytes per vector of one Schlomilch application,
    T*32*L + (2P+1)*8*L + 8*L with T = 2M(2P+1)."""
    L = params.n
    nb = len(scheme.blocks)
    T = 2 * params.m_terms * nb
    return T * 32 * L + nb * 8 * L + 8 * L


def hbm_peak():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            return float(json.load(f)["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)"
    except Exception:
        return 6650.0, "fallback (B200_PROFILING.md 6.65 TB/s)"


class ClockSampler:
    """nvidia-smi clocks / throttle reasons sampled during the timed region."""

    FIELDS = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.hw_slowdown,"
              "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
              "clocks_event_reasons.sw_power_cap")

    def __init__(self, index):
        self.index = index
        self.proc = None
        self.lines = []

    def start(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.index), "--query-gpu=" + self.FIELDS, "--format=csv,noheader,nounits",
                 "-lms", "100"], stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.thread = threading.Thread(target=self._read, daemon=True)
            self.thread.start()
        except Exception:
            self.proc = None

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def stop(self):
        if self.proc is None:
            return None
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except Exception:
            self.proc.kill()
        sm, mx, reasons = [], 0.0, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in self.lines:
            p = [x.strip() for x in ln.split(",")]
            if len(p) < 7:
                continue
            try:
                sm.append(float(p[0]))
                mx = max(mx, float(p[1]))
            except ValueError:
                continue
            for nm, v in zip(names, p[3:7]):
                if v.lower() == "active":
                    reasons.add(nm)
        if not sm:
            return None
        return {"sm_mhz": float(np.median(sm)), "sm_max_mhz": mx, "reasons": sorted(reasons), "samples": len(sm)}


def cpu_baseline_subprocess(n, timeout_s=240):
    """Time the oracle on ONE cfg2 vector in a single-threaded subprocess."""
    code = (
        "import os,sys,time,json,numpy as np;sys.path.insert(0,%r);"
        "from oracle import fht_oracle as O;import bench as B;"
        "c=B.make_inputs(%d,1,0)[0];p=O.plan_params(%d,%d,%r,%r);"
        "t=time.perf_counter();f=O.schlomilch(p,c);t=time.perf_counter()-t;"
        "np.save(%r,f);print(json.dumps({'seconds':t}))"
    ) % (ROOT, n, NU, n, EPS, GAMMA, os.path.join("/tmp", "fhtb_cpu_ref_%d.npy" % n))
    env = dict(os.environ, OPENBLAS_NUM_THREADS="1", OMP_NUM_THREADS="1", MKL_NUM_THREADS="1")
    try:
        r = subprocess.run([sys.executable, "-c", code], capture_output=True, text=True, timeout=timeout_s, env=env)
        sec = json.loads(r.stdout.strip().splitlines()[-1])["seconds"]
        ref = np.load(os.path.join("/tmp", "fhtb_cpu_ref_%d.npy" % n))
        return sec, ref
    except Exception as e:  # report, never fake
        return None, str(e)[:200]


def run_ours(args):
    import torch
    import torch.distributed as dist

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world > 1:
        os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)

    import paper_1501_01652_b200 as fh
    from paper_1501_01652_b200 import _lib
    from paper_1501_01652_b200.schlomilch import _grid

    n, batch = args.n, args.batch
    params = fh.select_params(NU, n, EPS, gamma=GAMMA)
    scheme = fh.build_partition(params)
    host = make_inputs(n, batch, rank)
    C = torch.from_numpy(host).to(dev)
    F = torch.zeros_like(C)
    grid = _grid(params.n, params.gamma, params.m_terms, scheme.blocks, scheme.mask_segments, [NU])
    reqs = [dict(vec=v, terms=[(NU, 1.0)]) for v in range(batch)]
    lib = _lib.load()
    st = torch.cuda.current_stream()

    def step():
        # one application, far + near field (the near field runs on its own
        # stream beside the far-field chunks inside the library)
        F.zero_()
        grid.apply(reqs, C, F, _lib.FHTB_FAR | _lib.FHTB_NEAR)

    def phases(n_rep):
        """far-only / near-only applications, CUDA-event timed (diagnostic,
        outside the timed region)"""
        ev = [torch.cuda.Event(enable_timing=True) for _ in range(3)]
        far, near = [], []
        for _ in range(n_rep):
            F.zero_()
            ev[0].record(st)
            grid.apply(reqs, C, F, _lib.FHTB_FAR)
            ev[1].record(st)
            grid.apply(reqs, C, F, _lib.FHTB_NEAR)
            ev[2].record(st)
            torch.cuda.synchronize()
            far.append(ev[0].elapsed_time(ev[1]))
            near.append(ev[1].elapsed_time(ev[2]))
        return float(np.mean(far)), float(np.mean(near))

    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize()
    t0, t1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    clk = ClockSampler(local)
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    clk.start()
    time.sleep(0.3)
    l0 = lib.fhtb_launch_count()
    t0.record(st)
    for k in range(args.steps):
        step()
    t1.record(st)
    torch.cuda.synchronize()
    l1 = lib.fhtb_launch_count()
    clocks = clk.stop()
    if world > 1:
        dist.barrier()
    ms = t0.elapsed_time(t1)
    if world > 1:
        t = torch.tensor([ms], device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms = float(t.item())
    ms_step = ms / args.steps
    value = batch * world / (ms_step / 1e3)

    # parity spot check of the timed output against the direct-summation
    # sample rows and (rank 0) the CPU oracle
    out = F.cpu().numpy()
    far_ms, near_ms = phases(max(2, min(args.steps, 5)))

    # end to end through the public API: pinned host in, host out
    if args.no_e2e:
        if rank == 0:
            print(json.dumps({"value": value, "ms_per_step": ms_step, "far_ms": far_ms, "near_ms": near_ms}))
        return
    pinned = torch.from_numpy(host).pin_memory()
    for _ in range(2):
        fh.schlomilch_fast(params, pinned)
    torch.cuda.synchronize()
    e2e_t = []
    for _ in range(max(1, min(args.steps, 5))):
        torch.cuda.synchronize()
        a = time.perf_counter()
        res = fh.schlomilch_fast(params, pinned)
        torch.cuda.synchronize()
        e2e_t.append(time.perf_counter() - a)
    e2e_s = float(np.median(e2e_t))
    if world > 1:
        t = torch.tensor([e2e_s], device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        e2e_s = float(t.item())
    assert np.array_equal(res.numpy(), out), "e2e result differs from the device-resident run"
    del pinned, res
    tasks = None if args.no_tasks else run_tasks(fh, dev, rank, world, max(2, min(args.steps, 5)), 2)

    if rank != 0:
        if world > 1:
            dist.destroy_process_group()
        return

    peak, peak_src = hbm_peak()
    # algorithmic bytes of the formulation actually executed (pruned side
    # blocks need no or a partial intermediate), and the unpruned SURVEY 8(d)
    # figure for reference
    bpv = lib.fhtb_grid_far_model_bytes(grid.handle)
    bpv_survey = model_bytes(params, scheme)
    achieved = bpv * batch / (far_ms / 1e3) / 1e9
    line = {
        "metric": METRIC,
        "value": value,
        "unit": UNIT,
        "n_gpus": world,
        "steps": args.steps,
        "warmup": args.warmup,
        "ms_per_step": ms_step,
        "higher_is_better": True,
        "scaling": "weak",
        "vs_baseline": None,
        "dtype": "f64",
        "data": "synthetic (seeded numpy PCG64, c_n = g_n/n, g ~ N(0,1))",
        "config": {"workload": "cfg2 Schlomilch nu=4 gamma=4 N=2^20 eps=1e-15", "N": n, "nu": NU,
                   "gamma": GAMMA, "eps": EPS, "batch_per_gpu": batch, "M": params.m_terms,
                   "P": params.partitions, "blocks": len(scheme.blocks), "near_field_entries": scheme.mask_size(),
                   "l2": "inputs 512 MiB/GPU > 126 MB L2; no flush", "parallelism": "dp%d (vector sharding)" % world},
        "phase_ms": {"far_field": far_ms, "near_field": near_ms,
                     "note": "far-only and near-only applications timed with CUDA events right after the "
                             "timed region; the timed step runs both in one application, the near field "
                             "on its own stream beside the far-field chunks"},
        "roofline": {"bound": "hbm", "kernel": "far field (pass 1 + pass 2 / column-generated pass 2 / row sums)",
                     "achieved": achieved, "peak": peak, "unit": "GB/s", "frac": achieved / peak,
                     "traffic": traffic_from_profile(), "model_bytes_per_vector": bpv,
                     "survey_model_bytes_per_vector": bpv_survey,
                     "survey_model_equivalent_gbs": bpv_survey * batch / (far_ms / 1e3) / 1e9,
                     "peak_source": peak_src,
                     "limiter_evidence": bounds_from_profile()},
        "e2e": {"value": batch * world / e2e_s, "unit": UNIT, "h2d_bytes_per_step": int(host.nbytes),
                "d2h_bytes_per_step": int(out.nbytes),
                "path": "schlomilch_fast(pinned CPU tensor) -> fhtb_apply_host: copies in/out overlapped with "
                        "the far field in tapered vector groups; median of %d calls" % max(1, min(args.steps, 5))},
        "gpu_launches": int(l1 - l0),
        "clocks": clocks,
        "tasks": tasks,
    }
    if world == 1 and not args.no_cpu:
        sec, ref = cpu_baseline_subprocess(n)
        if sec is not None:
            err = float(np.max(np.abs(out[0] - ref)))
            tol = 10 * EPS * float(np.abs(host[0]).sum())
            line["cpu_baseline"] = {"value": 1.0 / sec, "unit": UNIT, "cores": 1, "kind": "port",
                                    "sample": "1 full cfg2 vector (N=2^20, eps=1e-15), oracle/fht_oracle.py, "
                                              "1 thread, host cores of the GPU box",
                                    "seconds": sec}
            line["parity_vs_oracle"] = {"max_abs_err": err, "tol_10_eps_l1": tol, "ok": err <= tol}
        else:
            line["cpu_baseline"] = {"value": None, "unit": UNIT, "cores": 1, "kind": "port",
                                    "sample": "failed: " + str(ref)}
    print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()


def run_tasks(fh, dev, rank, world, steps, warmup):
    """The other BASELINE configs: FB (cfg3), DHT (cfg4) and cfg2 at the
    looser eps, device-resident, CUDA-event timed, max over ranks."""
    import torch
    import torch.distributed as dist
    out = {}
    st = torch.cuda.current_stream()
    peak, _ = hbm_peak()

    def timed(fn):
        for _ in range(warmup):
            fn()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()
        a.record(st)
        for _ in range(steps):
            fn()
        b.record(st)
        torch.cuda.synchronize()
        ms = a.elapsed_time(b) / steps
        if world > 1:
            t = torch.tensor([ms], device=dev)
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            ms = float(t.item())
        return ms

    def rng(kind, n, b):
        g = np.random.default_rng([SEED + 7, n, rank * 1000 + b])
        return g.uniform(-1.0, 1.0, n) if kind == "u" else g.standard_normal(n)

    from paper_1501_01652_b200.fourier_bessel import select_neumann_params
    from paper_1501_01652_b200.schlomilch import SchlomilchEngine, _m_terms
    def fb_task(n, B, eps, key, desc):
        roots = fh.bessel_roots_j0(n)
        C = torch.from_numpy(np.stack([rng("u", n, b) for b in range(B)])).to(dev)
        ms = timed(lambda: fh.fourier_bessel_eval(0, C, eps, roots=roots))
        q = select_neumann_params(eps)
        R = 2 * q.t_terms + q.k_terms - 2
        eng = SchlomilchEngine(n, -0.25, eps / R, range(q.k_terms))
        bpv = R * model_bytes(eng.params, eng.scheme)
        out[key] = {"config": desc, "transforms_per_s": B * world / (ms / 1e3), "ms_per_step": ms,
                    "model_bytes_per_vector": bpv, "model_frac_of_hbm": bpv * B / (ms / 1e3) / 1e9 / peak}

    def dht_task(n, B, eps, key, desc):
        plan = fh.dht_plan(n, eps)
        C = torch.from_numpy(np.stack([rng("n", n, b) for b in range(B)])).to(dev)
        st_ = {}
        fh.dht(plan, C[:1], stats=st_)
        ms = timed(lambda: fh.dht(plan, C))
        from paper_1501_01652_b200.dht import _shared
        eng = _shared(plan)["engine"]
        reqs = st_.get("schlomilch_evaluations", 0)
        T = 2 * eng.params.m_terms * len(eng.scheme.blocks)
        L2 = 1 << int(math.ceil(math.log2(2 * n - 1)))
        bpv = reqs * (T * 2 * 32 * L2 + len(eng.scheme.blocks) * 8 * n + 8 * n)
        out[key] = {"config": desc, "transforms_per_s": B * world / (ms / 1e3), "ms_per_step": ms,
                    "requests_per_vector": reqs, "model": "row-restricted chirp-z (SURVEY 8(d))",
                    "model_bytes_per_vector": bpv, "model_frac_of_hbm": bpv * B / (ms / 1e3) / 1e9 / peak}

    fb_task(2 ** 18, 16, 1e-12, "fb_cfg3", "Fourier-Bessel order 0, N=2^18, 16 vectors U[-1,1], eps=1e-12")
    dht_task(2 ** 16, 8, 1e-15, "dht_cfg4", "DHT order 0, N=2^16, 8 vectors N(0,1), eps=1e-15")
    # the metric's N = 2^20 for the other two tasks (BASELINE.json metric)
    fb_task(2 ** 20, 16, 1e-12, "fb_n2^20", "Fourier-Bessel order 0, N=2^20, 16 vectors U[-1,1], eps=1e-12")
    dht_task(2 ** 20, 4, 1e-15, "dht_n2^20", "DHT order 0, N=2^20, 4 vectors N(0,1), eps=1e-15")
    # cfg2 at the looser eps
    n, B = 2 ** 20, 64
    Cs = torch.from_numpy(make_inputs(n, B, rank)).to(dev)
    for eps in (1e-3, 1e-8):
        p = fh.select_params(NU, n, eps, gamma=GAMMA)
        ms = timed(lambda: fh.schlomilch_fast(p, Cs))
        bpv = model_bytes(p, fh.build_partition(p))
        out["cfg2_eps%g" % eps] = {"transforms_per_s": B * world / (ms / 1e3), "ms_per_step": ms,
                                   "model_bytes_per_vector": bpv,
                                   "model_frac_of_hbm": bpv * B / (ms / 1e3) / 1e9 / peak}
    return out


def bounds_from_profile():
    """Limiter evidence of the dominant far kernels (ncu --set full,
    tools/kernel_bounds.py): they run at ~75% of L1/TEX (shared-memory FFT
    exchanges) with DRAM at 30-36%, so HBM is not what bounds them."""
    p = os.path.join(ROOT, "profiles", "far_kernel_bounds.json")
    try:
        with open(p) as f:
            seen, out = set(), []
            for d in json.load(f)["launches"]:
                if d["kernel"] in seen:
                    continue
                seen.add(d["kernel"])
                out.append({k: d.get(k) for k in ("kernel", "l1tex_pct", "dram_pct", "issue_pct", "duration_us")})
            return out
    except Exception:
        return None


def traffic_from_profile():
    p = os.path.join(ROOT, "profiles", "traffic.json")
    try:
        with open(p) as f:
            t = json.load(f)
            return t.get("far_field_dram_bytes_per_vector", t.get("far_pass_pair_bytes_per_vector"))
    except Exception:
        return None


def _ref_worker(args):
    n, b = args
    from oracle import fht_oracle as O
    c = make_inputs(n, b + 1, 0)[b]
    p = O.plan_params(NU, n, EPS, GAMMA)
    t = time.perf_counter()
    O.schlomilch(p, c)
    return time.perf_counter() - t


def run_reference(args):
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    os.environ["OPENBLAS_NUM_THREADS"] = "1"
    import multiprocessing as mp
    cores = os.cpu_count() or 1
    ctx = mp.get_context("spawn")
    budget = args.ref_budget
    with ctx.Pool(cores, initializer=_ref_init) as pool:
        pool.map(_ref_warm, range(cores))          # untimed warm-up (imports, small case)
        times, steps = [], 0
        t_all = time.perf_counter()
        while steps < args.steps:
            a = time.perf_counter()
            pool.map(_ref_worker, [(args.n, b) for b in range(cores)])
            times.append(time.perf_counter() - a)
            steps += 1
            if time.perf_counter() - t_all + times[-1] > budget:
                break
    sec = float(np.mean(times))
    value = cores / sec
    line = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": int(os.environ.get("WORLD_SIZE", "1")),
        "steps": steps, "steps_requested": args.steps, "warmup": args.warmup, "ms_per_step": sec * 1e3,
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic (seeded numpy PCG64, c_n = g_n/n, g ~ N(0,1))", "impl": "reference",
        "config": {"workload": "cfg2 Schlomilch nu=4 gamma=4 N=2^20 eps=1e-15", "N": args.n, "nu": NU,
                   "gamma": GAMMA, "eps": EPS},
        "cpu_baseline": {"value": value, "unit": UNIT, "cores": cores, "kind": "port",
                         "sample": "each step: %d processes x 1 full cfg2 vector (oracle/fht_oracle.py, NumPy "
                                   "port of the reference; OPENBLAS_NUM_THREADS=1); steps capped at %ds of wall"
                                   % (cores, budget)},
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


def _ref_init():
    os.environ["OPENBLAS_NUM_THREADS"] = "1"
    sys.path.insert(0, ROOT)


def _ref_warm(i):
    from oracle import fht_oracle as O
    c = make_inputs(4096, 1, 0)[0]
    O.schlomilch(O.plan_params(NU, 4096, EPS, GAMMA), c)
    return i


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--n", type=int, default=N_DEF)
    ap.add_argument("--batch", type=int, default=BATCH)
    ap.add_argument("--no-cpu", action="store_true", help="skip the CPU oracle baseline leg")
    ap.add_argument("--ref-budget", type=float, default=150.0)
    ap.add_argument("--no-e2e", action="store_true", help="device-resident timing only (profiling runs)")
    ap.add_argument("--no-tasks", action="store_true", help="skip the FB/DHT/other-eps task timings")
    args = ap.parse_args()
    if args.warmup < 3 and args.impl == "ours":
        args.warmup = 3
    if args.impl == "reference":
        run_reference(args)
    else:
        run_ours(args)


if __name__ == "__main__":
    main()
