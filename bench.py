"""Benchmark: transforms/s of the fast Schlomilch/FB/DHT hot path on B200.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
                    [--workload cfg2|sweep|single24]

Headline workload (BASELINE.json configs[1], "cfg2"): Schlomilch expansion
nu=4, omega_n=(n+4)pi, r_k=k/N, N=2^20, 64 vectors c_n = g_n/n, g ~ N(0,1)
(seeded), eps=1e-15, fp64.  One step = one application of the partitioned
scheme (fused DCT-I/DST-I far field + DMMA near field) to the 64 vectors,
inputs resident in HBM (512 MiB, larger than the 126 MB L2, so no flush is
needed between steps).  With N GPUs every rank runs its own 64 vectors
(weak scaling, no data-path collective); value = all vectors / max-rank time.

--gpus N without WORLD_SIZE in the environment re-launches this script under
torch.distributed.run with N ranks (one per GPU, NCCL, 127.0.0.1).

Other workloads (BASELINE.json configs[4]):
  sweep     batch of 256 vectors SHARDED over the ranks (strong scaling):
            Schlomilch nu=0 and DHT cells; each cell is also timed on rank 0
            alone with the whole batch, so the line carries X_1, X_G and the
            efficiency X_G / (G X_1).
  single24  ONE N=2^24 Schlomilch transform (nu=0, eps=1e-15) distributed
            over the ranks: exchange="alltoall" (distributed four-step, NCCL
            all-to-all transpose) and exchange="pairs" (term-pair split, one
            all-reduce), each against the single-GPU result.

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


def setup_dist(args):
    """(world, rank, local, dev) of this process; NCCL over NVLink for N>1.
    NCCL_DEBUG=INFO goes to one file per rank (not stdout, which carries the
    JSON line) so the communicator's nRanks / NVLS lines can be reported."""
    import torch
    import torch.distributed as dist
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world != args.gpus:
        raise SystemExit("bench.py: --gpus %d but WORLD_SIZE=%d" % (args.gpus, world))
    if world > 1:
        os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
        os.environ.setdefault("NCCL_DEBUG", "INFO")
        os.environ.setdefault("NCCL_DEBUG_SUBSYS", "INIT,NVLS")
        os.environ.setdefault("NCCL_DEBUG_FILE", "/tmp/fhtb_nccl.%d.%s.log" % (rank, os.getpid()))
        if args.dry_run:
            dist.init_process_group("gloo")
        else:
            dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    if args.dry_run:
        return world, rank, local, torch.device("cpu")
    torch.cuda.set_device(local)
    return world, rank, local, torch.device("cuda", local)


def nccl_report():
    """Communicator lines of this rank's NCCL_DEBUG_FILE (nRanks, NVLS)."""
    path = os.environ.get("NCCL_DEBUG_FILE")
    if not path or not os.path.exists(path):
        return None
    lines = open(path, errors="replace").read().splitlines()
    comm = [ln.split("NCCL INFO", 1)[-1].strip() for ln in lines if "nRanks" in ln][:4]
    nvls = [ln.split("NCCL INFO", 1)[-1].strip() for ln in lines if "NVLS" in ln][:4]
    return {"file": path, "comm_lines": comm, "nvls_lines": nvls}


def max_over_ranks(x, world, dev):
    """max of a float over all ranks (the contract's max-over-ranks time)."""
    if world == 1:
        return float(x)
    import torch
    import torch.distributed as dist
    t = torch.tensor([float(x)], dtype=torch.float64, device=dev)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def barrier(world):
    if world > 1:
        import torch.distributed as dist
        dist.barrier()


def timed_region(fn, steps, warmup, world, dev, on_stream=None):
    """W untimed warm-ups, then K steps bracketed by barrier + synchronize on
    both sides, timed with CUDA events on the current stream; max over ranks."""
    import torch
    for _ in range(warmup):
        fn()
    torch.cuda.synchronize()
    st = torch.cuda.current_stream()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    barrier(world)
    torch.cuda.synchronize()
    a.record(st)
    for _ in range(steps):
        fn()
    b.record(st)
    torch.cuda.synchronize()
    barrier(world)
    return max_over_ranks(a.elapsed_time(b), world, dev) / steps


def dry_run(args, world, rank, dev):
    """CPU plumbing check of the launcher (gloo): shard ranges, barrier and
    max-over-ranks on a fake workload; prints the JSON line on rank 0."""
    import torch
    from paper_1501_01652_b200 import dist as fdist
    lo, hi = fdist.shard_range(256, rank, world)
    t = time.perf_counter()
    x = torch.arange(lo, hi, dtype=torch.float64).sum()
    ms = (time.perf_counter() - t) * 1e3
    ms = max_over_ranks(ms, world, dev)
    tot = torch.tensor([float(x), float(hi - lo)], dtype=torch.float64)
    if world > 1:
        import torch.distributed as dist
        dist.all_reduce(tot)
    if rank == 0:
        print(json.dumps({"dry_run": True, "n_gpus": world, "workload": args.workload, "ms": ms,
                          "items": int(tot[1]), "checksum": float(tot[0])}), flush=True)


def run_ours(args):
    import torch

    world, rank, local, dev = setup_dist(args)
    if args.dry_run:
        dry_run(args, world, rank, dev)
    elif args.workload == "sweep":
        run_sweep(args, world, rank, local, dev)
    elif args.workload == "single24":
        run_single(args, world, rank, local, dev)
    else:
        run_cfg2(args, world, rank, local, dev)
    if world > 1:
        import torch.distributed as dist
        dist.barrier()
        dist.destroy_process_group()


def kernel_roofline(kt, steps, peak, step_ms, kt_step=None, steps_step=1):
    """roofline.kernels[]: per kernel family, the EXCLUSIVE CUDA-event time of
    its launches (library option "serial": every launch on one stream in plan
    order, so a launch's events bracket that kernel alone), its share of the
    serial step, the algorithmic bytes it moved and the fraction of HBM peak.
    `ms_in_timed_step` is the same family's event time inside the timed region,
    where two chunks and the near field run concurrently on their own streams
    (kernels then share the SMs, so those times overlap and sum past the step)."""
    out = []
    tot = sum(v["ms"] for v in kt.values()) / steps
    f64 = (fp64_peaks() or {}).get("dfma_tflops")
    for name, v in sorted(kt.items(), key=lambda kv: -kv[1]["ms"]):
        ms = v["ms"] / steps
        gbs = v["bytes"] / (v["ms"] / 1e3) / 1e9 if v["ms"] > 0 else 0.0
        tfl = v.get("flops", 0.0) / (v["ms"] / 1e3) / 1e12 if v["ms"] > 0 else 0.0
        k = {"kernel": name, "ms_per_step": ms, "share_of_step": ms / tot if tot else None,
             "launches_per_step": v["launches"] / steps, "bytes_per_step": v["bytes"] / steps,
             "achieved_gbs": gbs, "frac": gbs / peak if v["bytes"] else None,
             # nominal FFT flops (5 n log2 n per executed transform) against the measured DFMA peak
             "fft_tflops": tfl if tfl else None,
             "frac_fp64": tfl / f64 if (tfl and f64) else None,
             "avg_launch_us": 1e3 * v["ms"] / max(1, v["launches"])}
        if kt_step is not None and name in kt_step:
            k["ms_in_timed_step"] = kt_step[name]["ms"] / steps_step
        out.append(k)
    return out


def serial_kernel_times(lib, _lib, fn, reps):
    """Per-family exclusive times: `reps` applications with the library's
    "serial" and "kernel_timing" options on (diagnostic, after the timed region)."""
    import torch
    _lib.check(lib.fhtb_set_option(b"serial", 1))
    try:
        fn()
        torch.cuda.synchronize()
        _lib.check(lib.fhtb_set_option(b"kernel_timing", 1))
        _lib.kernel_times()
        for _ in range(reps):
            fn()
        torch.cuda.synchronize()
        kt = _lib.kernel_times()
    finally:
        _lib.check(lib.fhtb_set_option(b"kernel_timing", 0))
        _lib.check(lib.fhtb_set_option(b"serial", 0))
    return kt


def run_cfg2(args, world, rank, local, dev):
    import torch

    import paper_1501_01652_b200 as fh
    from paper_1501_01652_b200 import _device, _lib
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

    def zero():
        _lib.call("fhtb_zero_rows", _device.ptr(F), F.stride(0), F.shape[0], F.shape[1], _device.stream_ptr())

    def step():
        # one application, far + near field (the near field runs on its own
        # stream beside the far-field chunks inside the library)
        zero()
        grid.apply(reqs, C, F, _lib.FHTB_FAR | _lib.FHTB_NEAR)

    def phases(n_rep):
        """far-only / near-only applications, CUDA-event timed (diagnostic,
        outside the timed region)"""
        ev = [torch.cuda.Event(enable_timing=True) for _ in range(3)]
        far, near = [], []
        for _ in range(n_rep):
            zero()
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
    barrier(world)
    torch.cuda.synchronize()
    clk.start()
    time.sleep(0.3)
    # per-kernel CUDA events inside the timed region (roofline.kernels[])
    _lib.check(lib.fhtb_set_option(b"kernel_timing", 1))
    _lib.kernel_times()
    l0 = lib.fhtb_launch_count()
    t0.record(st)
    for k in range(args.steps):
        step()
    t1.record(st)
    torch.cuda.synchronize()
    l1 = lib.fhtb_launch_count()
    kt = _lib.kernel_times()
    _lib.check(lib.fhtb_set_option(b"kernel_timing", 0))
    clocks = clk.stop()
    barrier(world)
    ms = max_over_ranks(t0.elapsed_time(t1), world, dev)
    ms_step = ms / args.steps
    value = batch * world / (ms_step / 1e3)

    out = F.cpu().numpy()
    far_ms, near_ms = phases(max(2, min(args.steps, 5)))
    n_ser = max(2, min(args.steps, 3))
    kt_ser = serial_kernel_times(lib, _lib, step, n_ser)

    if args.no_e2e:
        if rank == 0:
            print(json.dumps({"value": value, "ms_per_step": ms_step, "far_ms": far_ms, "near_ms": near_ms,
                              "kernels": kt_ser, "kernels_in_step": kt, "serial_steps": n_ser}))
        return
    # end to end through the public API: pinned host in, host out
    pinned = torch.from_numpy(host).pin_memory()
    e2e_s = e2e_time(lambda: fh.schlomilch_fast(params, pinned), args, world, dev)
    res = fh.schlomilch_fast(params, pinned)
    assert np.array_equal(res.numpy(), out), "e2e result differs from the device-resident run"
    # ... and the reference's own calling convention: numpy in, numpy out
    e2e_np_s = e2e_time(lambda: fh.schlomilch_fast(params, host), args, world, dev)
    assert np.array_equal(fh.schlomilch_fast(params, host), out), "numpy e2e result differs from the device-resident run"
    del pinned, res
    tasks = None if args.no_tasks else run_tasks(fh, dev, rank, world, max(2, min(args.steps, 5)), 2)

    if rank != 0:
        return

    peak, peak_src = hbm_peak()
    # algorithmic bytes of the formulation actually executed (pruned side
    # blocks need no or a partial intermediate), and the unpruned SURVEY 8(d)
    # figure for reference
    bpv = lib.fhtb_grid_far_model_bytes(grid.handle)
    bpv_survey = model_bytes(params, scheme)
    kernels = kernel_roofline(kt_ser, n_ser, peak, ms_step, kt, args.steps)
    far_k = [k for k in kernels if k["kernel"].startswith("far_") and k["bytes_per_step"] > 0]
    dom = max(far_k, key=lambda k: k["ms_per_step"])
    far_bytes = sum(k["bytes_per_step"] for k in far_k)
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
        "roofline": {"bound": "hbm", "kernel": dom["kernel"],
                     "achieved": dom["achieved_gbs"], "peak": peak, "unit": "GB/s",
                     "frac": dom["achieved_gbs"] / peak,
                     "traffic": traffic_from_profile(dom["kernel"]),
                     "fp64": {"achieved": dom.get("fft_tflops"), "peak": (fp64_peaks() or {}).get("dfma_tflops"),
                              "unit": "TFLOP/s", "frac": dom.get("frac_fp64"),
                              "note": "nominal FFT flops 5 n log2 n of the dominant kernel / measured DFMA peak; "
                                      "the far-field kernels are bound by the fp64 pipe and shared-memory "
                                      "bandwidth, not by HBM (DESIGN.md 3)"},
                     "how": "dominant kernel family (largest exclusive time): its algorithmic bytes (executed "
                            "formulation, DESIGN.md 3) / its CUDA-event time, launches serialised on one "
                            "stream (library option serial) over %d steps right after the timed region; "
                            "kernels[].ms_in_timed_step are the same events inside the timed region, where "
                            "concurrent chunks share the SMs" % n_ser,
                     "kernels": kernels,
                     "far_field": {"model_bytes_per_vector": bpv, "bytes_per_step": far_bytes,
                                   "frac_of_step": far_bytes / (ms_step / 1e3) / 1e9 / peak,
                                   "frac_far_only_call": bpv * batch / (far_ms / 1e3) / 1e9 / peak,
                                   "survey_model_bytes_per_vector": bpv_survey},
                     "peak_source": peak_src,
                     "fp64_peaks": fp64_peaks(),
                     "limiter_evidence": bounds_from_profile()},
        "e2e": {"value": batch * world / e2e_s, "unit": UNIT, "h2d_bytes_per_step": int(host.nbytes),
                "d2h_bytes_per_step": int(out.nbytes),
                "path": "schlomilch_fast(pinned CPU tensor) -> fhtb_apply_host: copies in/out overlapped with "
                        "the far field in tapered vector groups; median of %d calls" % max(1, min(args.steps, 5)),
                "numpy": {"value": batch * world / e2e_np_s, "unit": UNIT,
                          "path": "schlomilch_fast(numpy array) -> numpy array (the reference's calling "
                                  "convention): rows staged through pinned buffers in 8-vector chunks by two "
                                  "host threads, chunks alternating between two streams"}},
        "gpu_launches": int(l1 - l0),
        "clocks": clocks,
        "tasks": tasks,
    }
    if world > 1:
        line["nccl"] = nccl_report()
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


def e2e_time(fn, args, world, dev):
    """Median wall time of a public-API call with host buffers (copies in
    the timed region), max over ranks."""
    import torch
    for _ in range(2):
        fn()
    torch.cuda.synchronize()
    ts = []
    for _ in range(max(1, min(args.steps, 5))):
        barrier(world)
        torch.cuda.synchronize()
        a = time.perf_counter()
        fn()
        torch.cuda.synchronize()
        ts.append(time.perf_counter() - a)
    return max_over_ranks(float(np.median(ts)), world, dev)


def fp64_peaks():
    try:
        with open(os.path.join(ROOT, "profiles", "fp64_peak.json")) as f:
            d = json.load(f)
        return {"dfma_tflops": d["dfma"]["tflops"], "dmma_tflops": d["dmma"]["tflops"],
                "source": "profiles/fp64_peak.json (tools/fp64_peak.cu on this pool's B200)"}
    except Exception:
        return None


SWEEP_DEFAULT = "schl:10,schl:14,schl:20,dht:12,dht:16"


def run_sweep(args, world, rank, local, dev):
    """configs[4]: B vectors sharded over the ranks (strong scaling)."""
    import torch

    import paper_1501_01652_b200 as fh
    from paper_1501_01652_b200 import dist as fdist

    B = args.sweep_batch
    cells = []
    for item in (args.sweep or SWEEP_DEFAULT).split(","):
        task, lg = item.split(":")
        for eps in [float(e) for e in args.sweep_eps.split(",")]:
            cells.append((task, int(lg), eps))
    peak, _ = hbm_peak()
    res = []
    for task, lg, eps in cells:
        n = 1 << lg
        if task == "schl":
            p = fh.select_params(0, n, eps)
            fn_of = lambda C, p=p: (lambda: fh.schlomilch_fast(p, C))
        else:
            plan = fh.dht_plan(n, eps)
            fn_of = lambda C, plan=plan: (lambda: fh.dht(plan, C))
        lo, hi = fdist.shard_range(B, rank, world)
        rows = [np.random.default_rng([SEED, n, 1000 + b]).standard_normal(n) for b in range(lo, hi)]
        C = torch.from_numpy(np.stack(rows)).to(dev)
        ms_g = timed_region(fn_of(C), args.steps, max(3, args.warmup // 2), world, dev)
        x_g = B / (ms_g / 1e3)
        cell = {"task": task, "N": n, "eps": eps, "batch": B, "ms_per_step": ms_g, "transforms_per_s": x_g,
                "vectors_per_rank": [fdist.shard_range(B, r, world) for r in range(world)]}
        if world > 1:
            # X_1: rank 0 alone with the whole batch (other ranks wait)
            ms1 = 0.0
            if rank == 0:
                allrows = np.stack([np.random.default_rng([SEED, n, 1000 + b]).standard_normal(n)
                                    for b in range(B)])
                CA = torch.from_numpy(allrows).to(dev)
                ms1 = timed_region(fn_of(CA), args.steps, 2, 1, dev)
                del CA
            ms1 = max_over_ranks(ms1, world, dev)
            cell["x1_transforms_per_s"] = B / (ms1 / 1e3)
            cell["efficiency"] = x_g / (world * cell["x1_transforms_per_s"])
        res.append(cell)
        del C
        torch.cuda.empty_cache()
    if rank == 0:
        head = res[0]
        for c in res:
            if c["task"] == "schl" and c["N"] >= head["N"] and c["eps"] == 1e-15:
                head = c
        line = {"metric": "transforms/s, configs[4] sweep: batch %d sharded over %d GPU(s)" % (B, world),
                "value": head["transforms_per_s"], "unit": UNIT, "n_gpus": world, "steps": args.steps,
                "warmup": args.warmup, "ms_per_step": head["ms_per_step"], "higher_is_better": True,
                "scaling": "strong", "vs_baseline": None, "dtype": "f64",
                "data": "synthetic (seeded numpy PCG64, c ~ N(0,1))",
                "config": {"workload": "sweep", "headline_cell": "%s N=%d eps=%g" % (head["task"], head["N"],
                                                                                   head["eps"]),
                           "batch": B, "parallelism": "dp%d (batch sharding, no data-path collective)" % world},
                "cells": res}
        if world > 1:
            line["nccl"] = nccl_report()
        print(json.dumps(line), flush=True)


def run_single(args, world, rank, local, dev):
    """configs[4]: ONE N=2^24 transform distributed over the ranks."""
    import torch

    import paper_1501_01652_b200 as fh
    from paper_1501_01652_b200 import dist as fdist

    n, eps = args.single_n, 1e-15
    p = fh.select_params(0, n, eps)
    c = np.random.default_rng([SEED, n, 24]).standard_normal(n)
    C = torch.from_numpy(c).to(dev)
    ref = fh.schlomilch_fast(p, C)              # the plain single-GPU call
    tol = 10 * eps * float(np.abs(c).sum())
    out = {}
    for exchange in ("alltoall", "pairs"):
        fn = lambda: fdist.distributed_transform(fh.schlomilch_fast, p, C, exchange=exchange)
        ms = timed_region(fn, args.steps, 2, world, dev)
        got = fn()
        err = max_over_ranks(float((got - ref).abs().max()), world, dev)
        out[exchange] = {"ms": ms, "transforms_per_s": 1e3 / ms, "max_abs_err_vs_1gpu": err, "tol": tol,
                         "ok": err <= tol}
    if rank == 0:
        line = {"metric": "transforms/s, ONE N=2^%d Schlomilch transform (nu=0, eps=1e-15) over %d GPU(s)"
                          % (int(math.log2(n)), world),
                "value": out["alltoall"]["transforms_per_s"], "unit": UNIT, "n_gpus": world,
                "steps": args.steps, "warmup": args.warmup, "ms_per_step": out["alltoall"]["ms"],
                "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f64",
                "data": "synthetic (seeded numpy PCG64, c ~ N(0,1))",
                "config": {"workload": "single24", "N": n, "eps": eps,
                           "parallelism": "distributed four-step (NCCL all-to-all) vs term-pair split"},
                "exchanges": out}
        if world > 1:
            line["nccl"] = nccl_report()
        print(json.dumps(line), flush=True)


def run_tasks(fh, dev, rank, world, steps, warmup):
    """The other BASELINE configs: FB (cfg3), DHT (cfg4) and cfg2 at the
    looser eps, device-resident, CUDA-event timed, max over ranks.  Each
    task's HBM fraction uses the algorithmic bytes of the formulation the
    library executed (recorded per launch by the kernel timing), over the
    whole step time; kernels[] are exclusive times of a serialised application
    (serial_kernel_times)."""
    import torch
    from paper_1501_01652_b200 import _lib
    lib = _lib.load()
    out = {}
    peak, _ = hbm_peak()

    def timed(fn):
        for _ in range(warmup):
            fn()
        torch.cuda.synchronize()
        ms = timed_region(fn, steps, 0, world, dev)
        kt = serial_kernel_times(lib, _lib, fn, 2)
        return ms, kt

    def record(key, desc, B, ms, kt, extra=None):
        far_bytes = sum(v["bytes"] for k, v in kt.items() if k.startswith(("far_", "chirp_"))) / 2
        d = {"config": desc, "transforms_per_s": B * world / (ms / 1e3), "ms_per_step": ms,
             "executed_bytes_per_vector": far_bytes / B,
             "frac_of_hbm": far_bytes / (ms / 1e3) / 1e9 / peak,
             "kernels": kernel_roofline(kt, 2, peak, ms)}
        d.update(extra or {})
        out[key] = d

    def rng(kind, n, b):
        g = np.random.default_rng([SEED + 7, n, rank * 1000 + b])
        return g.uniform(-1.0, 1.0, n) if kind == "u" else g.standard_normal(n)

    def fb_task(n, B, eps, key, desc):
        roots = fh.bessel_roots_j0(n)
        C = torch.from_numpy(np.stack([rng("u", n, b) for b in range(B)])).to(dev)
        ms, kt = timed(lambda: fh.fourier_bessel_eval(0, C, eps, roots=roots))
        record(key, desc, B, ms, kt)

    def dht_task(n, B, eps, key, desc):
        plan = fh.dht_plan(n, eps)
        C = torch.from_numpy(np.stack([rng("n", n, b) for b in range(B)])).to(dev)
        st_ = {}
        fh.dht(plan, C[:1], stats=st_)
        ms, kt = timed(lambda: fh.dht(plan, C))
        record(key, desc, B, ms, kt, {"requests_per_vector": st_.get("schlomilch_evaluations", 0),
                                      "formulation": "row-restricted chirp-z (DESIGN.md 3)"})

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
        ms, kt = timed(lambda: fh.schlomilch_fast(p, Cs))
        record("cfg2_eps%g" % eps, "cfg2 at eps=%g" % eps, B, ms, kt)
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


def traffic_from_profile(kernel, batch=BATCH):
    """ncu dram__bytes_read.sum + dram__bytes_write.sum per step of the
    kernel family (profiles/traffic.json, tools/traffic.py), or None."""
    p = os.path.join(ROOT, "profiles", "traffic.json")
    try:
        with open(p) as f:
            t = json.load(f)
        v = t.get("per_family_dram_bytes_per_vector", {}).get(kernel)
        return None if v is None else v * batch
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


def relaunch(args):
    """--gpus N with no WORLD_SIZE: re-run this script under
    torch.distributed.run with N ranks on this node (127.0.0.1)."""
    import socket
    with socket.socket() as sk:
        sk.bind(("127.0.0.1", 0))
        port = sk.getsockname()[1]
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", str(args.gpus),
           "--master-addr", "127.0.0.1", "--master-port", str(port), os.path.abspath(__file__)] + sys.argv[1:]
    return subprocess.call(cmd)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--workload", default="cfg2", choices=["cfg2", "sweep", "single24"])
    ap.add_argument("--n", type=int, default=N_DEF)
    ap.add_argument("--batch", type=int, default=BATCH)
    ap.add_argument("--sweep", default="", help="cells task:log2N,... (default %s)" % SWEEP_DEFAULT)
    ap.add_argument("--sweep-eps", default="1e-15")
    ap.add_argument("--sweep-batch", type=int, default=256)
    ap.add_argument("--single-n", type=int, default=2 ** 24)
    ap.add_argument("--no-cpu", action="store_true", help="skip the CPU oracle baseline leg")
    ap.add_argument("--ref-budget", type=float, default=150.0)
    ap.add_argument("--no-e2e", action="store_true", help="device-resident timing only (profiling runs)")
    ap.add_argument("--no-tasks", action="store_true", help="skip the FB/DHT/other-eps task timings")
    ap.add_argument("--dry-run", action="store_true", help="launcher plumbing only (gloo, no GPU work)")
    args = ap.parse_args()
    if args.gpus < 1:
        raise SystemExit("--gpus must be >= 1")
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        sys.exit(relaunch(args))
    if args.warmup < 3 and args.impl == "ours":
        args.warmup = 3
    if args.impl == "reference":
        run_reference(args)
    else:
        run_ours(args)


if __name__ == "__main__":
    main()
