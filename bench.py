#!/usr/bin/env python
"""Benchmark of the precondition + sparsify + covariance hot path (BASELINE.json metric).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--workload c3] [--impl ours|reference]

One JSON line on rank 0. A "step" is one pass of the hot path over the workload's rows:
  covariance workloads (c1/c3/c4): K1a indices -> K1b gather (precondition + sample) -> K2 moments
                                   -> K3 covariance -> (N>1: one allreduce) -> K4 finalize
  kmeans workloads (c2/c5):        the Lloyd loop (max_iter iterations, stops on convergence)
                                   on the HBM-resident sketch, from seeded initial points
Compute defaults to f64: the drop-in sketch_stream's default and the reference's arithmetic
(bit-exact values). Scaling defaults to "strong": BASELINE's n is the whole job, sharded over
the N ranks with global column offsets. ``value`` is whole-job throughput with inputs resident
in HBM (larger than the 126 MB L2, so no flush is needed). ``e2e`` runs the same metric
through the public API from pinned host rows (H2D and the D2H of the result inside the timed
region). At N=1 the default run adds one line per other BASELINE config under "configs".
--impl reference times the reference CPU path on the host cores: the oracle port (C, all
threads) as the arm's value, and beside it the reference package itself (baseline/_ref).
"""

from __future__ import annotations

import argparse
import gc
import json
import os
import statistics
import subprocess
import sys
import tempfile
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

WORKLOADS = {
    # BASELINE.json configs; n is the whole job (strong scaling shards it over the ranks)
    "c1": dict(desc="C1 sparsified PCA p=256 m=25 (spiked rank-5)", p=256, n=20000, m=25, kind="cov", pcs=5),
    "c1big": dict(desc="C1 shape at steady state, n=2^24", p=256, n=1 << 24, m=25, kind="cov", pcs=5),
    "c2": dict(desc="C2 sparsified K-means p=512 m=26 K=10", p=512, n=200000, m=26, K=10, iters=20, kind="kmeans"),
    "c3": dict(desc="C3 large covariance p=1024 m=51 (spiked rank-10 + Student-t(3))", p=1024, n=1 << 24, m=51,
               kind="cov", pcs=0),
    "c4": dict(desc="C4 spiky covariance p=4096 m=82", p=4096, n=1 << 21, m=82, kind="cov", pcs=20),
    "c5": dict(desc="C5 sparsified K-means p=2048 m=102 K=100", p=2048, n=10_000_000, m=102, K=100, iters=10,
               kind="kmeans"),
}
SEED = 2026
MEASURED = os.path.join(ROOT, "MEASURED_PEAKS.json")
REF_PATH = os.path.join(ROOT, "baseline", "_ref")


def derive_seed(seed, tag):
    z = (seed ^ tag) & 0xFFFFFFFFFFFFFFFF
    M = 0xFFFFFFFFFFFFFFFF
    z = ((z ^ (z >> 30)) * 0xBF58476D1CE4E5B9) & M
    z = ((z ^ (z >> 27)) * 0x94D049BB133111EB) & M
    return z ^ (z >> 31)


def peaks():
    try:
        with open(MEASURED) as f:
            d = json.load(f)
        return float(d["hbm_gbs"]), "measured (MEASURED_PEAKS.json)"
    except Exception:
        return 6650.0, "fallback (B200_PROFILING.md)"


def metric_name(cfg):
    return "samples/s precondition+sparsify+covariance" if cfg["kind"] == "cov" else "K-means point-iters/s"


# ------------------------------------------------------------------ synthetic data
def _model(wl: str, rng):
    cfg = WORKLOADS[wl]
    p = cfg["p"]
    if wl.startswith("c1"):
        return np.linalg.qr(rng.standard_normal((p, 5)))[0], np.array([50.0, 40.0, 30.0, 20.0, 10.0])
    if wl == "c3":
        return np.linalg.qr(rng.standard_normal((p, 10)))[0], np.arange(100.0, 9.0, -10.0)
    if wl == "c4":
        return np.linalg.qr(rng.standard_normal((p, 20)))[0], np.linspace(20.0, 1.0, 20)
    K = cfg["K"]
    C = rng.standard_normal((p, K)) * (2.0 if wl == "c2" else 3.0)
    prob = np.full(K, 1.0 / K) if wl == "c2" else rng.dirichlet(np.ones(K))
    return C, prob


def gen_rows(wl: str, n: int, row0: int, device, torch):
    """(n, p) fp32 rows of workload wl, seeded per 2^18-row chunk of the global index."""
    cfg = WORKLOADS[wl]
    p = cfg["p"]
    X = torch.empty((n, p), dtype=torch.float32, device=device)
    g = torch.Generator(device=device)
    A, lam = _model(wl, np.random.default_rng(SEED))
    kmeans = wl in ("c2", "c5")
    if kmeans:
        Ct = torch.as_tensor(A.T.copy(), dtype=torch.float32, device=device)
        cdf = torch.as_tensor(np.cumsum(lam), dtype=torch.float64, device=device)
    else:
        B = torch.as_tensor((A * np.sqrt(lam)[None, :]).T.copy(), dtype=torch.float32, device=device)
    CH = 1 << 18
    for c0 in range(0, n, CH):
        c = min(CH, n - c0)
        g.manual_seed(SEED * 1000003 + (row0 + c0) // CH)
        if kmeans:
            u = torch.rand(c, generator=g, device=device, dtype=torch.float64)
            lab = torch.searchsorted(cdf, u).clamp_(max=cfg["K"] - 1)
            X[c0 : c0 + c] = Ct[lab] + torch.randn((c, p), generator=g, device=device)
            continue
        z = torch.randn((c, B.shape[0]), generator=g, device=device)
        sig = z @ B
        if wl == "c3":  # Student-t(3) scaled to unit variance: N / sqrt(chi2_3)
            num = torch.randn((c, p), generator=g, device=device)
            den = torch.randn((c, p), generator=g, device=device).square_()
            den += torch.randn((c, p), generator=g, device=device).square_()
            den += torch.randn((c, p), generator=g, device=device).square_()
            sig += num / den.sqrt_()
        elif wl == "c4":  # 8 spikes of +-50 per sample + N(0, 0.01)
            sig += 0.1 * torch.randn((c, p), generator=g, device=device)
            pos = torch.randint(0, p, (c, 8), generator=g, device=device)
            sgn = torch.randint(0, 2, (c, 8), generator=g, device=device).float() * 100.0 - 50.0
            sig.scatter_(1, pos, sgn)
        else:
            sig += torch.randn((c, p), generator=g, device=device)
        X[c0 : c0 + c] = sig
    return X


def gen_rows_np(wl: str, n: int, seed: int = SEED) -> np.ndarray:
    """The same generative model in numpy (the reference arm uses no GPU)."""
    cfg = WORKLOADS[wl]
    p = cfg["p"]
    rng = np.random.default_rng(seed)
    A, lam = _model(wl, np.random.default_rng(SEED))
    if wl in ("c2", "c5"):
        lab = np.minimum(np.searchsorted(np.cumsum(lam), rng.random(n)), cfg["K"] - 1)
        return (A.T[lab] + rng.standard_normal((n, p))).astype(np.float32)
    X = rng.standard_normal((n, len(lam))) @ (A * np.sqrt(lam)[None, :]).T
    if wl == "c3":
        X += rng.standard_normal((n, p)) / np.sqrt(rng.chisquare(3, (n, p)))
    elif wl == "c4":
        X += 0.1 * rng.standard_normal((n, p))
        rows = np.repeat(np.arange(n), 8)
        X[rows, rng.integers(0, p, n * 8)] = rng.choice([-50.0, 50.0], n * 8)
    else:
        X += rng.standard_normal((n, p))
    return X.astype(np.float32)


# ------------------------------------------------------------------ clocks
class ClockSampler:
    """SM clock and throttle reasons sampled DURING the timed region.

    NVML polled every 5 ms from a thread (short regions still get samples), else the
    recipe's ``nvidia-smi --query-gpu=... -lms 100`` line."""

    REASONS = (("hw_slowdown", "nvmlClocksEventReasonHwSlowdown"),
               ("hw_thermal_slowdown", "nvmlClocksEventReasonHwThermalSlowdown"),
               ("sw_thermal_slowdown", "nvmlClocksEventReasonSwThermalSlowdown"),
               ("sw_power_cap", "nvmlClocksEventReasonSwPowerCap"))

    def __init__(self, index: int, pci_bus_id: str = None):
        self.index, self.pci = index, pci_bus_id
        self.rows, self.max_mhz, self.source = [], None, None
        self.stop = threading.Event()
        self.thread = self.p = self.f = None

    def _nvml_loop(self, N, h):
        bits = [(name, getattr(N, const, 0)) for name, const in self.REASONS]
        while not self.stop.is_set():
            try:
                sm = N.nvmlDeviceGetClockInfo(h, N.NVML_CLOCK_SM)
                r = N.nvmlDeviceGetCurrentClocksEventReasons(h)
                util = N.nvmlDeviceGetUtilizationRates(h).gpu
                self.rows.append((float(sm), [name for name, b in bits if r & b], int(util)))
            except Exception:
                pass
            self.stop.wait(0.005)

    def __enter__(self):
        try:
            import pynvml as N

            N.nvmlInit()
            h = (N.nvmlDeviceGetHandleByPciBusId(self.pci) if self.pci else N.nvmlDeviceGetHandleByIndex(self.index))
            self.max_mhz = float(N.nvmlDeviceGetMaxClockInfo(h, N.NVML_CLOCK_SM))
            self.source = "nvml 5 ms"
            self.thread = threading.Thread(target=self._nvml_loop, args=(N, h), daemon=True)
            self.thread.start()
            return self
        except Exception:
            self.thread = None
        try:
            self.f = tempfile.NamedTemporaryFile("w+", suffix=".csv", delete=False)
            self.p = subprocess.Popen(
                ["nvidia-smi", f"--id={self.index}",
                 "--query-gpu=clocks.sm,clocks.max.sm,clocks_event_reasons.active,"
                 "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
                 "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap,utilization.gpu",
                 "--format=csv,noheader,nounits", "-lms", "100"], stdout=self.f, stderr=subprocess.DEVNULL)
            self.source = "nvidia-smi 100 ms"
        except Exception:
            self.p = None
        return self

    def __exit__(self, *a):
        if self.thread is not None:
            self.stop.set()
            self.thread.join()
        if self.p is not None:
            self.p.terminate()
            self.p.wait()
            self.f.flush()
            self.f.seek(0)
            for r in (r.split(",") for r in self.f.read().strip().splitlines()):
                if len(r) < 8 or not r[0].strip().replace(".", "").isdigit():
                    continue
                if self.max_mhz is None and r[1].strip().replace(".", "").isdigit():
                    self.max_mhz = float(r[1])
                util = int(r[7]) if r[7].strip().isdigit() else 1
                self.rows.append((float(r[0]), [self.REASONS[i][0] for i in range(4) if r[3 + i].strip() == "Active"],
                                  util))

    def summary(self):
        if not self.rows:
            return {"sm_mhz": None, "sm_max_mhz": self.max_mhz, "reasons": ["unavailable"], "source": self.source}
        busy = [r for r in self.rows if r[2] > 0] or self.rows
        return {"sm_mhz": statistics.median(r[0] for r in busy), "sm_max_mhz": self.max_mhz,
                "reasons": sorted({x for r in busy for x in r[1]}), "samples": len(busy), "source": self.source}


# ------------------------------------------------------------------ CPU legs (oracle port)
def cpu_cov_rate(rows: np.ndarray, cfg, nthreads: int, min_seconds: float = 10.0):
    """The oracle port (oracle/, C, all host threads) on a bounded row sample: samples/s."""
    from oracle import oracle as O

    p, m = cfg["p"], cfg["m"]
    ss, ms = derive_seed(SEED, 0xD5), derive_seed(SEED, 0x5A)
    done, t0 = 0, time.perf_counter()
    while True:
        idx, val = O.sketch(rows, p, O.HADAMARD, ss, ms, m, col0=0, nthreads=nthreads)
        O.cov_finalize(O.cov_acc(idx, val, p, nthreads), p, m, rows.shape[0])
        O.mean_acc(idx, val, p)
        done += rows.shape[0]
        el = time.perf_counter() - t0
        if el >= min_seconds:
            return done / el, el


def cpu_kmeans_rate(rows: np.ndarray, cfg, nthreads: int, min_seconds: float = 10.0):
    """The oracle port's Lloyd iteration (assign + update) on a bounded sample: point-iters/s."""
    from oracle import oracle as O

    p, m, K = cfg["p"], cfg["m"], cfg["K"]
    ss, ms = derive_seed(SEED, 0xD5), derive_seed(SEED, 0x5A)
    idx, val = O.sketch(rows, p, O.HADAMARD, ss, ms, m, nthreads=nthreads)
    chosen = np.random.default_rng(SEED).choice(rows.shape[0], K, replace=False)
    mu = O.init_centers(idx, val, chosen, p)
    pts, t0 = 0, time.perf_counter()
    while True:
        labels, _ = O.kmeans_assign(idx, val, mu, nthreads)
        mu, _, _ = O.kmeans_update(idx, val, labels, mu)
        pts += rows.shape[0]
        el = time.perf_counter() - t0
        if el >= min_seconds:
            return pts / el, el


def cpu_baseline(wl: str, cfg, seconds: float = 10.0, rows: np.ndarray = None):
    nthreads = os.cpu_count() or 1
    sample = min(cfg["n"], 1 << 16)
    if rows is None:
        rows = gen_rows_np(wl, sample)
    if cfg["kind"] == "cov":
        rate, el = cpu_cov_rate(rows, cfg, nthreads, seconds)
        unit = "samples/s"
    else:
        rate, el = cpu_kmeans_rate(rows, cfg, nthreads, seconds)
        unit = "point-iters/s"
    return {"value": rate, "unit": unit, "cores": nthreads, "kind": "port",
            "sample": f"{rows.shape[0]} rows of {wl} (same generative model), repeated for {el:.1f} s"}


# ------------------------------------------------------------------ the reference package itself
def _ref_import():
    if REF_PATH not in sys.path:
        sys.path.insert(0, REF_PATH)
    import sketchpipe  # noqa: F401  (baseline/_ref: pip install --target of /root/reference/pkg)

    return sketchpipe


def _ref_shard_worker(args):
    """One process of the sharded reference run: its column range with GLOBAL offsets
    (sketch.py:211-220 primitives), then its partial W W^T (estimators.py:59-61)."""
    wl, g0, g1, seconds = args
    sp = _ref_import()
    from sketchpipe.sketch import SparseSketch
    from sketchpipe.transform import precondition_columns

    cfg = WORKLOADS[wl]
    spec = sp.PreconditionSpec.create("hadamard", cfg["p"], sign_seed=derive_seed(SEED, 0xD5))
    plan = sp.SamplingPlan(derive_seed(SEED, 0x5A), spec.p_pad, cfg["m"])
    X = gen_rows_np(wl, g1 - g0, seed=SEED + g0).T.astype(np.float64)
    done, t0 = 0, time.perf_counter()
    while True:
        Y = precondition_columns(X, spec)
        idx = plan.indices_block(g0, g1)
        val = np.take_along_axis(Y.T, idx.astype(np.int64), axis=1)
        W = SparseSketch(spec=spec, n=g1 - g0, indices=idx, values=val, plan=plan).to_csc()
        (W @ W.T).toarray()
        np.bincount(idx.ravel(), weights=val.ravel(), minlength=spec.p_pad)
        done += g1 - g0
        if time.perf_counter() - t0 >= seconds:
            return done, time.perf_counter() - t0


def python_reference(wl: str, cfg, seconds: float = 12.0):
    """sketchpipe itself: (i) one process through its public API,
    (ii) one process per host core on global column ranges."""
    try:
        sp = _ref_import()
    except Exception as e:  # noqa: BLE001
        return {"unavailable": f"baseline/_ref not importable: {e}"}
    out = {"package": "sketchpipe (baseline/_ref, unmodified)"}
    p, m = cfg["p"], cfg["m"]
    spec = sp.PreconditionSpec.create("hadamard", p, sign_seed=derive_seed(SEED, 0xD5))
    plan = sp.SamplingPlan(derive_seed(SEED, 0x5A), spec.p_pad, m)
    ns = min(cfg["n"], 8192 if p >= 2048 else 16384)
    X = gen_rows_np(wl, ns).T.astype(np.float64)
    if cfg["kind"] == "cov":
        done, t0 = 0, time.perf_counter()
        while True:
            sk = sp.sketch_stream(sp.ArraySource(X), spec, plan)
            sp.estimate_covariance(sk)
            sp.estimate_mean(sk)
            done += ns
            if time.perf_counter() - t0 >= seconds:
                break
        el = time.perf_counter() - t0
        out["single_process"] = {"value": done / el, "unit": "samples/s", "cores": 1,
                                 "sample": f"{ns} columns, sketch_stream + estimate_covariance + estimate_mean"}
        procs = os.cpu_count() or 1
        import multiprocessing as mpc

        per = max(1024, ns // 2)
        ctx = mpc.get_context("fork")
        with ctx.Pool(procs) as pool:
            res = pool.map(_ref_shard_worker, [(wl, r * per, (r + 1) * per, seconds) for r in range(procs)])
        el = max(r[1] for r in res)
        out["multi_process"] = {"value": sum(r[0] for r in res) / el, "unit": "samples/s", "cores": procs,
                                "sample": f"{procs} processes x {per} columns (global offsets), "
                                          "precondition_columns + indices_block + gather + W W^T"}
    else:
        from sketchpipe.cluster import _SparseOps

        sk = sp.sketch_stream(sp.ArraySource(X), spec, plan)
        ops = _SparseOps(sk)
        K = cfg["K"]
        mu = ops.init_centers(np.random.default_rng(SEED).choice(ns, K, replace=False))
        pts, t0 = 0, time.perf_counter()
        while True:
            labels, d2min = ops.assign(mu)
            mu, empty = ops.update(labels, mu, K)
            pts += ns
            if time.perf_counter() - t0 >= seconds:
                break
        el = time.perf_counter() - t0
        out["single_process"] = {"value": pts / el, "unit": "point-iters/s", "cores": 1,
                                 "sample": f"{ns} points, _SparseOps assign + update (cluster.py:231-241)"}
    return out


def run_reference(args, cfg):
    nthreads = os.cpu_count() or 1
    sample = min(cfg["n"], 1 << 16 if cfg["p"] >= 1024 else 1 << 17)
    rows = gen_rows_np(args.workload, sample)
    per_step, per_step_s = [], []
    for i in range(args.warmup + args.steps):
        if cfg["kind"] == "cov":
            rate, el = cpu_cov_rate(rows, cfg, nthreads, min_seconds=0.0)
        else:
            rate, el = cpu_kmeans_rate(rows, cfg, nthreads, min_seconds=0.0)
        if i >= args.warmup:
            per_step.append(rate)
            per_step_s.append(el)
    value = statistics.median(per_step)
    unit = "samples/s" if cfg["kind"] == "cov" else "point-iters/s"
    desc = f"{sample} rows of {args.workload}, oracle port (C) with {nthreads} threads"
    out = {
        "impl": "reference", "metric": metric_name(cfg), "value": value, "unit": unit, "n_gpus": args.gpus,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * statistics.median(per_step_s),
        "higher_is_better": True, "scaling": args.scaling,
        "vs_baseline": None, "dtype": "f64", "data": "synthetic (numpy, same generative model)",
        "config": {"workload": args.workload, "desc": cfg["desc"], "p": cfg["p"], "m": cfg["m"]},
        "cpu_baseline": {"value": value, "unit": unit, "cores": nthreads, "kind": "port", "sample": desc},
        "e2e": {"value": value, "unit": unit, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    if not args.no_python_ref:
        out["python_reference"] = python_reference(args.workload, cfg)
    return out


# ------------------------------------------------------------------ our arm
class Ctx:
    def __init__(self, torch, tdist, skc, lib, sdist, dev, rank, world, local, hbm_peak, peak_src):
        self.torch, self.tdist, self.skc, self.lib, self.sdist = torch, tdist, skc, lib, sdist
        self.dev, self.rank, self.world, self.local = dev, rank, world, local
        self.hbm_peak, self.peak_src = hbm_peak, peak_src
        self.L = lib.lib()
        try:
            pr = torch.cuda.get_device_properties(dev)
            self.pci = f"{pr.pci_domain_id:08X}:{pr.pci_bus_id:02X}:{pr.pci_device_id:02X}.0"
        except Exception:
            self.pci = None

    def barrier(self):
        if self.world > 1:
            self.tdist.barrier()
        self.torch.cuda.synchronize()

    def max_over_ranks(self, v: float) -> float:
        t = self.torch.tensor([v], dtype=self.torch.float64, device=self.dev)
        if self.world > 1:
            self.tdist.all_reduce(t, op=self.tdist.ReduceOp.MAX)
        return float(t.item())


def shard(cfg, ctx, scaling):
    if scaling == "weak":
        return cfg["n"], ctx.rank * cfg["n"], cfg["n"] * ctx.world
    c0, c1 = ctx.sdist.shard_bounds(cfg["n"], ctx.rank, ctx.world)
    return c1 - c0, c0, cfg["n"]


def profiled_kernel(workload, n, stage, compute):
    """dram read+write bytes per launch of the stage's kernel from the committed ncu capture
    (profiles/<wl>_ncu_full.json, tools/ncu_summary.py) when it was taken at this size and
    compute type, else None."""
    names = {"indices": "indices_kernel", "gather": "gtma::gather_tma_kernel", "covariance": "cov_flat_kernel",
             "moments": "moments_kernel"}
    path = os.path.join(ROOT, "profiles", f"{workload}_ncu_full.json")
    try:
        with open(path) as f:
            d = json.load(f)
        if f"n=2^{int(np.log2(n))}" not in d["config"] or (1 << int(np.log2(n))) != n or compute not in d["config"]:
            return None
        for k, v in d["kernels"].items():
            if k.startswith(names.get(stage, "?")):
                return v
    except Exception:
        return None
    return None


def profiled_traffic(workload, n, stage, compute):
    v = profiled_kernel(workload, n, stage, compute)
    return v.get("traffic_bytes") if v else None


def lloyd_traffic(workload, n):
    """DRAM read+write bytes per Lloyd iteration (the K-means roofline's 'launch') from the committed
    ncu launch list (profiles/<wl>_ncu_lloyd.json, tools/ncu_iter_traffic.py) taken at this n, else None."""
    try:
        with open(os.path.join(ROOT, "profiles", f"{workload}_ncu_lloyd.json")) as f:
            d = json.load(f)
        return d["dram_bytes_per_iteration"] if int(d["points"]) == int(n) else None
    except Exception:
        return None


def cov_line(ctx, wl, args, steps, warmup, compute, sampler="oracle", clocks=True):
    """HBM-resident covariance pass (K1a..K4), stage-timed with CUDA events on the stream."""
    torch, skc, lib = ctx.torch, ctx.skc, ctx.lib
    cfg = WORKLOADS[wl]
    n, col0, n_glob = shard(cfg, ctx, args.scaling)
    p, m = cfg["p"], cfg["m"]
    X = gen_rows(wl, n, col0, ctx.dev, torch)
    spec = skc.PreconditionSpec.create("hadamard", p, sign_seed=derive_seed(SEED, 0xD5))
    plan = skc.SamplingPlan(derive_seed(SEED, 0x5A), spec.p_pad, m)
    vcode = lib.F32 if compute == "f32" else lib.F64
    vdt = torch.float32 if compute == "f32" else torch.float64
    idx = torch.empty((n, m), dtype=torch.int32, device=ctx.dev)
    val = torch.empty((n, m), dtype=vdt, device=ctx.dev)
    mom = skc.estimators.Moments.zeros(p, True, ctx.dev)
    C = torch.empty((p, p), dtype=torch.float64, device=ctx.dev)
    L = ctx.L
    ws1 = lib.workspace(L.skc_moments_workspace(n, m, p), ctx.dev)
    ws2 = lib.workspace(L.skc_cov_workspace(n, m, p), ctx.dev)
    st = lib.stream_ptr(ctx.dev)
    names = ["indices", "gather", "moments", "covariance", "combine+finalize"]

    def step(ev):
        mom.packed.zero_()
        ev[0].record()
        # the sketch as the two kernels skc_sketch runs: K1a indices (oracle keys or Philox), K1b gather
        if sampler == "philox":
            lib.call("skc_indices_philox", plan.master_seed, col0, n, p, m, idx.data_ptr(), st)
        else:
            lib.call("skc_indices", plan.master_seed, col0, n, p, m, idx.data_ptr(), st)
        ev[1].record()
        lib.call("skc_sketch_given", X.data_ptr(), lib.F32, p, n, p, p, 0, spec.sign_seed, m, vcode,
                 idx.data_ptr(), val.data_ptr(), vcode, st)
        ev[2].record()
        lib.call("skc_moments", idx.data_ptr(), val.data_ptr(), vcode, n, m, p, mom.acc.data_ptr(),
                 mom.stats.data_ptr(), ws1.data_ptr(), ws1.numel(), st)
        ev[3].record()
        lib.call("skc_cov_accumulate", idx.data_ptr(), val.data_ptr(), vcode, n, m, p, mom.stats.data_ptr(),
                 mom.tri.data_ptr(), ws2.data_ptr(), ws2.numel(), st)
        ev[4].record()
        ctx.sdist.combine_moments(mom.acc, mom.stats, mom.tri, n, n_total=n_glob)  # one allreduce (N > 1)
        lib.call("skc_cov_finalize", mom.tri.data_ptr(), p, m, n_glob, C.data_ptr(), st)
        ev[5].record()

    def mk():
        return [torch.cuda.Event(enable_timing=True) for _ in range(6)]

    for _ in range(warmup):
        step(mk())
        # warm-up passes end with a synchronise, as a chunked pipeline's passes do: K3 tunes its band
        # plan from the previous launch's per-band cycle counts (read back without blocking), so
        # the previous launch has to have finished when the next one is enqueued
        torch.cuda.synchronize()
    ctx.barrier()
    evs = [mk() for _ in range(steps)]
    launches0 = L.skc_launch_count()
    clk = ClockSampler(ctx.local, ctx.pci) if clocks else None
    if clk:
        clk.__enter__()
    t0 = torch.cuda.Event(enable_timing=True)
    t1 = torch.cuda.Event(enable_timing=True)
    ctx.barrier()
    t0.record()
    for k in range(steps):
        step(evs[k])
    t1.record()
    ctx.barrier()
    if clk:
        clk.__exit__()
    launches = L.skc_launch_count() - launches0
    ms_step = ctx.max_over_ranks(t0.elapsed_time(t1) / steps)
    stage_ms = {nm: sum(e[i].elapsed_time(e[i + 1]) for e in evs) / steps for i, nm in enumerate(names)}
    vsz = 4 if compute == "f32" else 8
    # algorithmic bytes per sample: the index kernel writes idx; the gather reads the row and idx
    # and writes values; K2 / K3 read the (index, value) pairs
    unit_bytes = {"indices": 4 * m, "gather": 4 * p + 4 * m + vsz * m, "moments": (4 + vsz) * m,
                  "covariance": (4 + vsz) * m, "combine+finalize": 0}
    dom = max((k for k in unit_bytes if unit_bytes[k] > 0), key=lambda k: stage_ms[k])
    dom_bytes = unit_bytes[dom] * n
    achieved = dom_bytes / (stage_ms[dom] * 1e-3) / 1e9
    roofline = {"bound": "hbm", "kernel": dom, "achieved": achieved, "peak": ctx.hbm_peak, "unit": "GB/s",
                "frac": achieved / ctx.hbm_peak, "traffic": profiled_traffic(wl, n, dom, compute),
                "peak_source": ctx.peak_src, "algorithmic_bytes_per_launch": dom_bytes,
                "bytes_per_sample": {k: v for k, v in unit_bytes.items() if v}}
    per_stage = {k: {"ms": stage_ms[k], "algorithmic_GBps": unit_bytes[k] * n / (stage_ms[k] * 1e-3) / 1e9,
                     "frac_hbm": unit_bytes[k] * n / (stage_ms[k] * 1e-3) / 1e9 / ctx.hbm_peak}
                 for k in unit_bytes if unit_bytes[k] > 0 and stage_ms[k] > 0}
    upd = n * m * (m + 1) / 2 / (stage_ms["covariance"] * 1e-3)
    per_stage["covariance"]["pair_updates_per_s"] = upd
    per_stage["covariance"]["frac_of_measured_smem_atomic_peak"] = upd / 1.355e12  # tools/microbench/mb_dsmem
    # K3's binding resource is the shared-memory pipe (profiles/round2/notes.md): its busy fraction
    # from the committed ncu capture of this shape, when there is one
    kc = profiled_kernel(wl, n, "covariance", compute)
    if kc and "l1tex_busy_pct" in kc:
        per_stage["covariance"]["smem_pipe_busy_frac_ncu"] = kc["l1tex_busy_pct"] / 100.0
    roofline["stages"] = per_stage
    roofline["pass_frac_hbm"] = (4 * p + (4 + vsz) * m) * (n / (ms_step * 1e-3)) / 1e9 / ctx.hbm_peak
    out = {"metric": metric_name(cfg), "value": n_glob / (ms_step * 1e-3), "unit": "samples/s",
           "ms_per_step": ms_step, "dtype": compute, "stages_ms": stage_ms, "roofline": roofline,
           "gpu_launches": int(launches), "rows_per_gpu": n, "global_rows": n_glob}
    if clk:
        out["clocks"] = clk.summary()
    if cfg.get("pcs"):
        # the host eigensolve of the PCA configs (north_star: handed back to the host), reported apart
        Ch = C.cpu().numpy()
        t = time.perf_counter()
        skc.top_eigenvectors(Ch, cfg["pcs"])
        out["host_eigensolve_ms"] = (time.perf_counter() - t) * 1e3
    del X, idx, val
    torch.cuda.empty_cache()
    return out


def release_pinned(torch):
    """Return cached pinned host blocks to the OS (the host caching allocator keeps freed
    blocks; the e2e legs pin up to 82 GB each on a 196 GB host)."""
    gc.collect()
    try:
        torch._C._host_emptyCache()
    except Exception:  # noqa: BLE001
        pass


def pinned_rows(ctx, wl, n, col0):
    torch = ctx.torch
    host = torch.empty((n, WORKLOADS[wl]["p"]), dtype=torch.float32, pin_memory=True)
    CH = 1 << 20
    for r in range(0, n, CH):
        c = min(CH, n - r)
        host[r : r + c].copy_(gen_rows(wl, c, col0 + r, ctx.dev, torch))
    return host


def cov_e2e(ctx, wl, args, compute, reps=3):
    """The same metric through the public API from pinned host rows: stream_moments (the
    native chunk loop, H2D of chunk k+1 overlapped with chunk k's kernels), one allreduce,
    covariance_from_moments, D2H of the p x p result, timed on the host wall clock."""
    skc = ctx.skc
    cfg = WORKLOADS[wl]
    n, col0, n_glob = shard(cfg, ctx, args.scaling)
    p, m = cfg["p"], cfg["m"]
    spec = skc.PreconditionSpec.create("hadamard", p, sign_seed=derive_seed(SEED, 0xD5))
    plan = skc.SamplingPlan(derive_seed(SEED, 0x5A), spec.p_pad, m)
    host = pinned_rows(ctx, wl, n, col0)
    src = skc.RowSource(host, chunk_cols=1 << 16)

    def one():
        mom = skc.stream_moments(src, spec, plan, compute=compute, col0=col0)
        ctx.sdist.combine_moments(mom.acc, mom.stats, mom.tri, mom.n, n_total=n_glob)
        return skc.covariance_from_moments(mom, p, m, n_glob).cpu().numpy()

    one()
    ctx.barrier()
    w0 = time.perf_counter()
    for _ in range(reps):
        one()
    ctx.barrier()
    e_ms = ctx.max_over_ranks((time.perf_counter() - w0) * 1e3 / reps)
    del host, src
    release_pinned(ctx.torch)
    return {"value": n_glob / (e_ms * 1e-3), "unit": "samples/s", "h2d_bytes_per_step": n * p * 4,
            "d2h_bytes_per_step": p * p * 8, "ms_per_step": e_ms, "rows_per_gpu": n, "compute": compute,
            "api": "stream_moments(RowSource(pinned host rows)) + combine_moments + covariance_from_moments "
                   "-> host (p, p): per-chunk sketch, moments and covariance overlapped with the next chunk's H2D"}


def kmeans_line(ctx, wl, args, steps, warmup, clocks=True):
    """Lloyd loop on the HBM-resident f64 sketch (reference arithmetic, bit-exact labels)."""
    torch, skc = ctx.torch, ctx.skc
    cfg = WORKLOADS[wl]
    n, col0, n_glob = shard(cfg, ctx, args.scaling)
    p, m, K = cfg["p"], cfg["m"], cfg["K"]
    X = gen_rows(wl, n, col0, ctx.dev, torch)
    spec = skc.PreconditionSpec.create("hadamard", p, sign_seed=derive_seed(SEED, 0xD5))
    plan = skc.SamplingPlan(derive_seed(SEED, 0x5A), spec.p_pad, m)
    sk = skc.sketch_stream(skc.RowSource(X), spec, plan, compute="f64", col0=col0)
    del X
    torch.cuda.empty_cache()
    ops = skc.SketchKMeans(sk)
    chosen = np.random.default_rng(SEED).choice(n_glob, K, replace=False)  # global seeded points
    mu0 = ctx.sdist.init_centers_global(ops, chosen)
    torch.cuda.synchronize()
    t = time.perf_counter()
    ops.prepare(K)  # once per sketch: transposed lists (+ tensor-core entries), reported apart
    torch.cuda.synchronize()
    prep_ms = ctx.max_over_ranks((time.perf_counter() - t) * 1e3)
    for _ in range(warmup):
        ops.lloyd(mu0, cfg["iters"])
    ctx.barrier()
    L = ctx.L
    launches0 = L.skc_launch_count()
    clk = ClockSampler(ctx.local, ctx.pci) if clocks else None
    if clk:
        clk.__enter__()
    t0 = torch.cuda.Event(enable_timing=True)
    t1 = torch.cuda.Event(enable_timing=True)
    ctx.barrier()
    t0.record()
    its = 0
    for _ in range(steps):
        its += ops.lloyd(mu0, cfg["iters"])[3]
    t1.record()
    ctx.barrier()
    if clk:
        clk.__exit__()
    launches = L.skc_launch_count() - launches0
    ms_step = ctx.max_over_ranks(t0.elapsed_time(t1) / steps)
    it_step = its / steps
    rate = n_glob * it_step / (ms_step * 1e-3)
    ub = 12 * m + 4  # f64 sketch row (idx + value) + a label, per point-iteration
    gbs = ub * n * it_step / (ms_step * 1e-3) / 1e9
    out = {"metric": metric_name(cfg), "value": rate, "unit": "point-iters/s", "ms_per_step": ms_step,
           "iterations_per_step": it_step, "dtype": "f64", "prep_ms": prep_ms, "gpu_launches": int(launches),
           "rows_per_gpu": n, "global_rows": n_glob,
           "roofline": {"bound": "hbm", "kernel": "lloyd iteration (assign + partials + centres)",
                        "achieved": gbs, "peak": ctx.hbm_peak, "unit": "GB/s", "frac": gbs / ctx.hbm_peak,
                        "traffic": lloyd_traffic(wl, n), "peak_source": ctx.peak_src, "bytes_per_point_iter": ub}}
    if clk:
        out["clocks"] = clk.summary()
    del sk, ops
    torch.cuda.empty_cache()
    return out


def kmeans_e2e(ctx, wl, args, reps=None):
    """sparsified_kmeans(pinned host rows of this rank's shard, init=seeded global points) ->
    host labels and centres; under torchrun every rank passes its shard (col0 from rank order)
    and the public API runs the sharded Lloyd loop. Host wall clock, max over ranks."""
    torch, skc = ctx.torch, ctx.skc
    cfg = WORKLOADS[wl]
    n, col0, n_glob = shard(cfg, ctx, args.scaling)
    p, m, K = cfg["p"], cfg["m"], cfg["K"]
    host = pinned_rows(ctx, wl, n, col0)
    chosen = np.random.default_rng(SEED).choice(n_glob, K, replace=False)
    src = skc.RowSource(host, chunk_cols=1 << 16)
    gamma = m / p

    def one():
        r = skc.sparsified_kmeans(src, K, gamma, max_iter=cfg["iters"], seed=SEED, init=chosen, col0=col0)
        return r.diagnostics["iterations"]

    one()
    # each call timed on its own (host wall clock, max over ranks); the median call is reported,
    # since a single host-side hiccup on a fresh box can multiply one call's time (tools/km_e2e_probe.py)
    if reps is None:
        reps = 3 if n <= 1_000_000 else 1
    times, its = [], 0
    for _ in range(reps):
        ctx.barrier()
        w0 = time.perf_counter()
        its = one()
        ctx.barrier()
        times.append(ctx.max_over_ranks(time.perf_counter() - w0))
    el = float(np.median(times)) * reps
    del host, src
    release_pinned(torch)
    return {"value": n_glob * its * reps / el, "unit": "point-iters/s", "h2d_bytes_per_step": n * p * 4,
            "d2h_bytes_per_step": n * 8 + p * K * 8, "ms_per_step": el * 1e3 / reps,
            "iterations_per_step": its, "rows_per_gpu": n, "calls_timed": reps, "statistic": "median call",
            "api": "sparsified_kmeans(RowSource(pinned host rows), K, gamma, init=seeded points): H2D + sketch + "
                   "Lloyd loop + host labels and centres (per-rank bytes; every rank its shard)"}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--workload", default="c3", choices=sorted(WORKLOADS))
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--n", type=int, default=None, help="override the whole-job row count")
    ap.add_argument("--compute", default="f64", choices=["f32", "f64"])
    ap.add_argument("--scaling", default="strong", choices=["strong", "weak"])
    ap.add_argument("--sampler", default="oracle", choices=["oracle", "philox"],
                    help="oracle: the reference's index rule (bit-exact, headline); philox: north_star's Philox sampler")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--no-configs", action="store_true", help="skip the per-config lines of the other workloads")
    ap.add_argument("--no-secondary", action="store_true", help="skip the philox / f32 secondaries")
    ap.add_argument("--no-python-ref", action="store_true")
    args = ap.parse_args()
    if args.n:
        WORKLOADS[args.workload]["n"] = args.n
    cfg = dict(WORKLOADS[args.workload])

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))

    if args.impl == "reference":
        if rank == 0:
            print(json.dumps(run_reference(args, cfg)), flush=True)
        return

    import torch
    import torch.distributed as tdist

    # one process per GPU; SKC_DIST_BACKEND=gloo (with fewer GPUs than ranks, ranks share devices)
    # exercises the multi-rank path on a single-GPU box -- a code check, not a timing
    backend = os.environ.get("SKC_DIST_BACKEND", "nccl")
    local_dev = local % max(1, torch.cuda.device_count())
    torch.cuda.set_device(local_dev)
    dev = torch.device("cuda", local_dev)
    if world > 1:
        os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
        if backend == "nccl":
            tdist.init_process_group("nccl", device_id=dev)
        else:
            tdist.init_process_group(backend)
    import paper_1511_00152_b200 as skc
    from paper_1511_00152_b200 import _lib
    from paper_1511_00152_b200 import dist as sdist

    hbm_peak, peak_src = peaks()
    ctx = Ctx(torch, tdist, skc, _lib, sdist, dev, rank, world, local_dev, hbm_peak, peak_src)
    wl = args.workload
    if cfg["kind"] == "cov":
        line = cov_line(ctx, wl, args, args.steps, args.warmup, args.compute, args.sampler)
    else:
        line = kmeans_line(ctx, wl, args, args.steps, args.warmup)
    out = {"metric": line["metric"], "value": line["value"], "unit": line["unit"], "n_gpus": world,
           "steps": args.steps, "warmup": args.warmup, "ms_per_step": line["ms_per_step"], "higher_is_better": True,
           "scaling": args.scaling, "vs_baseline": None, "dtype": line["dtype"],
           "data": "synthetic (seeded, device-generated; BASELINE.json generator shapes)",
           "config": {"workload": wl, "desc": cfg["desc"], "p": cfg["p"], "m": cfg["m"],
                      "rows_per_gpu": line["rows_per_gpu"], "global_rows": line["global_rows"],
                      "sampler": args.sampler, "parallelism": f"dp{world}",
                      "l2": "inputs larger than L2 (no flush needed)" if line["rows_per_gpu"] * cfg["p"] * 4 > 126e6
                      else "inputs fit L2"}}
    for k in ("stages_ms", "roofline", "gpu_launches", "clocks", "prep_ms", "iterations_per_step",
              "host_eigensolve_ms"):
        if k in line:
            out[k] = line[k]
    if cfg["kind"] == "cov" and not args.no_secondary:
        # north_star's Philox sampler and the f32 fast path, same shapes and timing (not bit-exact
        # to the reference: uniform m-subsets / fp32 values; pinned to their own oracles)
        ph = cov_line(ctx, wl, args, max(1, min(args.steps, 5)), 1, args.compute, "philox", clocks=False)
        out["philox_mode"] = {k: ph[k] for k in ("value", "unit", "ms_per_step", "stages_ms")}
        f32 = cov_line(ctx, wl, args, max(1, min(args.steps, 5)), 1, "f32", args.sampler, clocks=False)
        out["fast_mode_f32"] = {k: f32[k] for k in ("value", "unit", "ms_per_step", "stages_ms")}
        out["fast_mode_f32"]["gather_frac_hbm"] = f32["roofline"]["stages"]["gather"]["frac_hbm"]
    if not args.no_e2e:
        if cfg["kind"] == "cov":
            out["e2e"] = cov_e2e(ctx, wl, args, args.compute)
        else:
            out["e2e"] = kmeans_e2e(ctx, wl, args)
    if rank == 0 and world == 1 and not args.no_cpu:
        out["cpu_baseline"] = cpu_baseline(wl, cfg)

    # the other BASELINE configs, one line each (N=1 default run)
    if world == 1 and wl == "c3" and not args.no_configs:
        out["configs"] = {}
        for other in ("c1", "c2", "c4", "c5"):
            oc = WORKLOADS[other]
            gc.collect()
            torch.cuda.empty_cache()
            try:
                if oc["kind"] == "cov":
                    ln = cov_line(ctx, other, args, args.steps, args.warmup, args.compute, "oracle", clocks=False)
                else:
                    ln = kmeans_line(ctx, other, args, max(2, args.steps // 2), 1, clocks=False)
                ln["config"] = {"workload": other, "desc": oc["desc"], "p": oc["p"], "m": oc["m"], "n": oc["n"]}
                out["configs"][other] = ln
                if not args.no_e2e:
                    ln["e2e"] = (cov_e2e(ctx, other, args, args.compute) if oc["kind"] == "cov"
                                 else kmeans_e2e(ctx, other, args))
                if not args.no_cpu:
                    ln["cpu_baseline"] = cpu_baseline(other, oc, seconds=5.0)
            except Exception as e:  # noqa: BLE001  (one config failing must not lose the headline)
                out["configs"].setdefault(other, {})["error"] = f"{type(e).__name__}: {str(e)[:200]}"
                release_pinned(torch)
            torch.cuda.empty_cache()

    if rank == 0:
        print(json.dumps(out), flush=True)
    if world > 1:
        tdist.destroy_process_group()


if __name__ == "__main__":
    main()
