#!/usr/bin/env python
"""Benchmark of the precondition + sparsify + covariance hot path (BASELINE.json metric).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--workload c3] [--impl ours|reference]

One JSON line on rank 0. A "step" is one pass of the hot path over one batch:
  covariance workloads (c1/c3/c4): K1 sketch -> K2 moments -> K3 covariance -> K4 finalize
                                   over the whole HBM-resident sample set
  kmeans workloads (c2/c5):        the Lloyd loop (max_iter iterations, stops early on
                                   convergence) on the HBM-resident sketch
``value`` is whole-job throughput with inputs resident in HBM. ``e2e`` runs the same
metric through the public API (sketch_stream(RowSource(pinned host rows)) ->
estimate_covariance, so H2D and D2H happen inside the timed region). Inputs are larger
than the 126 MB L2, so no L2 flush is needed. --impl reference times the reference CPU
path, the oracle port in C (``oracle/``), on all host cores over a bounded sample.
"""

from __future__ import annotations

import argparse
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
    # BASELINE.json configs; n is per GPU (weak scaling)
    "c1": dict(desc="C1 sparsified PCA p=256 m=25 (spiked rank-5)", p=256, n=20000, m=25, kind="cov"),
    "c1big": dict(desc="C1 shape at steady state, n=2^24", p=256, n=1 << 24, m=25, kind="cov"),
    "c2": dict(desc="C2 sparsified K-means p=512 m=26 K=10", p=512, n=200000, m=26, K=10, iters=20, kind="kmeans"),
    "c3": dict(desc="C3 large covariance p=1024 m=51 (spiked rank-10 + Student-t(3))", p=1024, n=1 << 24, m=51,
               kind="cov"),
    "c4": dict(desc="C4 spiky covariance p=4096 m=82", p=4096, n=1 << 21, m=82, kind="cov"),
    "c5": dict(desc="C5 sparsified K-means p=2048 m=102 K=100", p=2048, n=10_000_000, m=102, K=100, iters=10,
               kind="kmeans"),
}
SEED = 2026
MEASURED = os.path.join(ROOT, "MEASURED_PEAKS.json")


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


# ------------------------------------------------------------------ synthetic data
def gen_rows(wl: str, n: int, row0: int, device, torch):
    """(n, p) fp32 rows of workload wl, seeded per 2^18-row chunk of the global index."""
    cfg = WORKLOADS[wl]
    p = cfg["p"]
    X = torch.empty((n, p), dtype=torch.float32, device=device)
    g = torch.Generator(device=device)
    rng = np.random.default_rng(SEED)
    if wl.startswith("c1"):
        U = np.linalg.qr(rng.standard_normal((p, 5)))[0]
        lam = np.array([50.0, 40.0, 30.0, 20.0, 10.0])
    elif wl == "c3":
        U = np.linalg.qr(rng.standard_normal((p, 10)))[0]
        lam = np.arange(100.0, 9.0, -10.0)
    elif wl == "c4":
        U = np.linalg.qr(rng.standard_normal((p, 20)))[0]
        lam = np.linspace(20.0, 1.0, 20)
    else:
        K = cfg["K"]
        C = rng.standard_normal((p, K)) * (2.0 if wl == "c2" else 3.0)
        if wl == "c2":
            prob = np.full(K, 1.0 / K)
        else:
            prob = rng.dirichlet(np.ones(K))
        Ct = torch.as_tensor(C.T.copy(), dtype=torch.float32, device=device)
        cdf = torch.as_tensor(np.cumsum(prob), dtype=torch.float64, device=device)
    if not wl.startswith("c2") and not wl.startswith("c5"):
        B = torch.as_tensor((U * np.sqrt(lam)[None, :]).T.copy(), dtype=torch.float32, device=device)
    CH = 1 << 18
    for c0 in range(0, n, CH):
        c = min(CH, n - c0)
        g.manual_seed(SEED * 1000003 + (row0 + c0) // CH)
        if wl in ("c2", "c5"):
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


# ------------------------------------------------------------------ clocks
class ClockSampler:
    def __init__(self, index: int):
        self.index = index
        self.f = tempfile.NamedTemporaryFile("w+", suffix=".csv", delete=False)
        self.p = None

    def __enter__(self):
        try:
            self.p = subprocess.Popen(
                ["nvidia-smi", f"--id={self.index}",
                 "--query-gpu=clocks.sm,clocks.max.sm,clocks_event_reasons.active,"
                 "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
                 "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap,utilization.gpu",
                 "--format=csv,noheader,nounits", "-lms", "100"], stdout=self.f, stderr=subprocess.DEVNULL)
        except Exception:
            self.p = None
        return self

    def __exit__(self, *a):
        if self.p is not None:
            self.p.terminate()
            self.p.wait()

    def summary(self):
        self.f.flush()
        self.f.seek(0)
        rows = [r.split(",") for r in self.f.read().strip().splitlines() if r.count(",") >= 7]
        if not rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unavailable"]}
        busy = [r for r in rows if r[7].strip().isdigit() and int(r[7]) > 0] or rows
        sm = [float(r[0]) for r in busy if r[0].strip().replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for r in busy for i in range(4) if r[3 + i].strip() == "Active"})
        return {"sm_mhz": statistics.median(sm) if sm else None,
                "sm_max_mhz": float(rows[0][1]) if rows[0][1].strip().replace(".", "").isdigit() else None,
                "reasons": reasons, "samples": len(busy)}


# ------------------------------------------------------------------ CPU baseline (oracle port)
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
    from oracle import oracle as O

    p, m, K = cfg["p"], cfg["m"], cfg["K"]
    ss, ms = derive_seed(SEED, 0xD5), derive_seed(SEED, 0x5A)
    idx, val = O.sketch(rows, p, O.HADAMARD, ss, ms, m, nthreads=nthreads)
    chosen = np.random.default_rng(SEED).choice(rows.shape[0], K, replace=False)
    mu = O.init_centers(idx, val, chosen, p)
    pts, t0 = 0, time.perf_counter()
    while True:
        labels, d2 = O.kmeans_assign(idx, val, mu, nthreads)
        mu, _, _ = O.kmeans_update(idx, val, labels, mu)
        pts += rows.shape[0]
        el = time.perf_counter() - t0
        if el >= min_seconds:
            return pts / el, el


# ------------------------------------------------------------------ reference arm
def run_reference(args, cfg):
    nthreads = os.cpu_count() or 1
    sample = min(cfg["n"], 1 << 16 if cfg["p"] >= 1024 else 1 << 17)
    rng = np.random.default_rng(SEED)
    rows = rng.standard_normal((sample, cfg["p"])).astype(np.float32)
    per_step = []
    for i in range(args.warmup + args.steps):
        if cfg["kind"] == "cov":
            rate, _ = cpu_cov_rate(rows, cfg, nthreads, min_seconds=0.0)
        else:
            rate, _ = cpu_kmeans_rate(rows, cfg, nthreads, min_seconds=0.0)
        if i >= args.warmup:
            per_step.append(rate)
    value = statistics.median(per_step)
    unit = "samples/s" if cfg["kind"] == "cov" else "point-iters/s"
    desc = f"{sample} rows of {args.workload}, oracle port (C) with {nthreads} threads"
    return {
        "impl": "reference", "metric": metric_name(cfg), "value": value, "unit": unit, "n_gpus": args.gpus,
        "steps": args.steps, "warmup": args.warmup, "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": {"workload": args.workload, "desc": cfg["desc"], "p": cfg["p"], "m": cfg["m"]},
        "cpu_baseline": {"value": value, "unit": unit, "cores": nthreads, "kind": "port", "sample": desc},
        "e2e": {"value": value, "unit": unit, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }


def profiled_traffic(workload, n, stage):
    """dram read+write bytes per launch of the stage's kernel, from the committed ncu capture
    (profiles/<wl>_ncu_full.json, written by tools/ncu_summary.py) when it was taken at this
    exact size, else None."""
    names = {"indices": "indices_kernel", "gather": "gather_kernel", "covariance": "cov_band_kernel",
             "moments": "moments_kernel"}
    path = os.path.join(ROOT, "profiles", f"{workload}_ncu_full.json")
    try:
        with open(path) as f:
            d = json.load(f)
        if f"n=2^{int(np.log2(n))}" not in d["config"] or (1 << int(np.log2(n))) != n:
            return None
        for k, v in d["kernels"].items():
            if k.startswith(names.get(stage, "?")):
                return v.get("traffic_bytes")
    except Exception:
        return None
    return None


def kmeans_secondary(wl, dev, torch, skc, hbm_peak, runs=2):
    """The Lloyd loop of a K-means config (sketch HBM-resident, seeded initial points), device-timed."""
    c = WORKLOADS[wl]
    X = gen_rows(wl, c["n"], 0, dev, torch)
    spec = skc.PreconditionSpec.create("hadamard", c["p"], sign_seed=derive_seed(SEED, 0xD5))
    plan = skc.SamplingPlan(derive_seed(SEED, 0x5A), spec.p_pad, c["m"])
    sk = skc.sketch_stream(skc.RowSource(X), spec, plan, compute="f64")
    del X
    torch.cuda.empty_cache()
    ops = skc.SketchKMeans(sk)
    mu0 = ops.init_centers(np.random.default_rng(SEED).choice(c["n"], c["K"], replace=False))
    ops.lloyd(mu0, c["iters"])  # warm-up: builds the transposed sketch and the tensor-core entries
    its, el = 0, 0.0
    for _ in range(runs):
        _, _, _, it_done, secs = ops.lloyd(mu0, c["iters"])
        its += it_done
        el += secs
    rate = c["n"] * its / el
    gbs = (8 * c["m"] + 4) * rate / 1e9  # algorithmic bytes per point-iteration: the sketch row + a label
    return {"metric": "K-means point-iters/s", "value": rate, "iterations_per_run": its / runs,
            "ms_per_run": el * 1e3 / runs, "desc": c["desc"],
            "roofline": {"bound": "hbm", "achieved": gbs, "peak": hbm_peak, "unit": "GB/s", "frac": gbs / hbm_peak},
            "note": "Lloyd loop on the HBM-resident f64 sketch, exact reference arithmetic (bit-identical labels)"}


def metric_name(cfg):
    if cfg["kind"] == "cov":
        return "samples/s precondition+sparsify+covariance"
    return "K-means point-iters/s"


# ------------------------------------------------------------------ our arm
def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--workload", default="c3", choices=sorted(WORKLOADS))
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--n", type=int, default=None, help="override rows per GPU")
    ap.add_argument("--compute", default="f64", choices=["f32", "f64"])
    ap.add_argument("--sampler", default="oracle", choices=["oracle", "philox"],
                    help="oracle: the reference's index rule (bit-exact, headline); philox: north_star's Philox sampler")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--no-kmeans", action="store_true")
    ap.add_argument("--no-philox", action="store_true", help="skip the Philox-sampler secondary measurement")
    ap.add_argument("--no-c5", action="store_true", help="skip the C5 K-means secondary measurement")
    args = ap.parse_args()
    cfg = dict(WORKLOADS[args.workload])
    if args.n:
        cfg["n"] = args.n

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))

    if args.impl == "reference":
        if rank == 0:
            print(json.dumps(run_reference(args, cfg)), flush=True)
        return

    import torch
    import torch.distributed as tdist

    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if world > 1:
        os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
        tdist.init_process_group("nccl", device_id=dev)
    import paper_1511_00152_b200 as skc
    from paper_1511_00152_b200 import _lib
    from paper_1511_00152_b200 import dist as sdist

    L = _lib.lib()
    hbm_peak, peak_src = peaks()
    n = cfg["n"]
    p, m = cfg["p"], cfg["m"]
    col0 = rank * n
    X = gen_rows(args.workload, n, col0, dev, torch)
    spec = skc.PreconditionSpec.create("hadamard", p, sign_seed=derive_seed(SEED, 0xD5))
    plan = skc.SamplingPlan(derive_seed(SEED, 0x5A), spec.p_pad, m)
    torch.cuda.synchronize()

    def barrier():
        if world > 1:
            tdist.barrier()
        torch.cuda.synchronize()

    stage_names, stage_ms = [], {}
    result = {}
    if cfg["kind"] == "cov":
        vcode = _lib.F32 if args.compute == "f32" else _lib.F64
        vdt = torch.float32 if args.compute == "f32" else torch.float64
        idx = torch.empty((n, m), dtype=torch.int32, device=dev)
        val = torch.empty((n, m), dtype=vdt, device=dev)
        acc = torch.zeros(p, dtype=torch.float64, device=dev)
        stats = torch.zeros(3, dtype=torch.float64, device=dev)
        tri = torch.zeros(p * (p + 1) // 2, dtype=torch.float64, device=dev)
        C = torch.empty((p, p), dtype=torch.float64, device=dev)
        ws1 = _lib.workspace(L.skc_moments_workspace(n, m, p), dev)
        ws2 = _lib.workspace(L.skc_cov_workspace(n, m, p), dev)
        st = _lib.stream_ptr(dev)
        ev = [torch.cuda.Event(enable_timing=True) for _ in range(6)]
        # the sketch as its two kernels (what skc_sketch runs internally), timed apart so the
        # roofline can name the dominant kernel: K1a indices (oracle keys or Philox), K1b gather
        stage_names = ["indices", "gather", "moments", "covariance", "finalize"]
        sampler = args.sampler

        def step(record):
            acc.zero_()
            stats.zero_()
            tri.zero_()
            if record:
                ev[0].record()
            if sampler == "philox":
                _lib.call("skc_indices_philox", plan.master_seed, col0, n, p, m, idx.data_ptr(), st)
            else:
                _lib.call("skc_indices", plan.master_seed, col0, n, p, m, idx.data_ptr(), st)
            if record:
                ev[1].record()
            _lib.call("skc_sketch_given", X.data_ptr(), _lib.F32, p, n, p, p, 0, spec.sign_seed, m, vcode,
                      idx.data_ptr(), val.data_ptr(), vcode, st)
            if record:
                ev[2].record()
            _lib.call("skc_moments", idx.data_ptr(), val.data_ptr(), vcode, n, m, p, acc.data_ptr(), stats.data_ptr(),
                      ws1.data_ptr(), ws1.numel(), st)
            if record:
                ev[3].record()
            _lib.call("skc_cov_accumulate", idx.data_ptr(), val.data_ptr(), vcode, n, m, p, stats.data_ptr(),
                      tri.data_ptr(), ws2.data_ptr(), ws2.numel(), st)
            if record:
                ev[4].record()
            n_tot = sdist.combine_moments(acc, stats, tri, n)
            _lib.call("skc_cov_finalize", tri.data_ptr(), p, m, n_tot, C.data_ptr(), st)
            if record:
                ev[5].record()

        for _ in range(args.warmup):
            step(False)
        barrier()
        launches0 = L.skc_launch_count()
        sums = [0.0] * len(stage_names)
        with ClockSampler(local) as clk:
            t0 = torch.cuda.Event(enable_timing=True)
            t1 = torch.cuda.Event(enable_timing=True)
            barrier()
            t0.record()
            for _ in range(args.steps):
                step(True)
                torch.cuda.synchronize()
                for i in range(len(stage_names)):
                    sums[i] += ev[i].elapsed_time(ev[i + 1])
            t1.record()
            barrier()
        launches = L.skc_launch_count() - launches0
        ms_total = t0.elapsed_time(t1)
        stage_ms = {k: sums[i] / args.steps for i, k in enumerate(stage_names)}
        ms_step = ms_total / args.steps
        vsz = 4 if args.compute == "f32" else 8
        # algorithmic bytes per sample: indices write idx; gather reads the row and idx, writes values
        unit_bytes = {"indices": 4 * m, "gather": 4 * p + 4 * m + vsz * m, "moments": (4 + vsz) * m,
                      "covariance": (4 + vsz) * m, "finalize": 0}
        total_samples = n * world
        unit = "samples/s"
        metric = metric_name(cfg)
        work_units = total_samples
    else:
        K, iters_max = cfg["K"], cfg["iters"]
        sk = skc.sketch_stream(skc.RowSource(X), spec, plan, compute="f64", col0=col0)
        ops = skc.SketchKMeans(sk)
        chosen = np.random.default_rng(SEED).choice(n, K, replace=False)
        mu0 = ops.init_centers(chosen)  # seeded points of rank 0's shard, the same centres on every rank
        if world > 1:
            tdist.broadcast(mu0, src=0)
        for _ in range(args.warmup):
            ops.lloyd(mu0, iters_max)
        barrier()
        launches0 = L.skc_launch_count()
        with ClockSampler(local) as clk:
            t0 = torch.cuda.Event(enable_timing=True)
            t1 = torch.cuda.Event(enable_timing=True)
            barrier()
            t0.record()
            its = 0
            for _ in range(args.steps):
                _, _, _, it_done, _ = ops.lloyd(mu0, iters_max)
                its += it_done
            t1.record()
            barrier()
        launches = L.skc_launch_count() - launches0
        ms_total = t0.elapsed_time(t1)
        ms_step = ms_total / args.steps
        stage_names = ["lloyd"]
        stage_ms = {"lloyd": ms_step}
        unit_bytes = {"lloyd": (8 * m + 4) * its / args.steps}
        unit = "point-iters/s"
        metric = metric_name(cfg)
        work_units = n * world * its / args.steps
        total_samples = n * world

    # max over ranks
    t = torch.tensor([ms_step], dtype=torch.float64, device=dev)
    if world > 1:
        tdist.all_reduce(t, op=tdist.ReduceOp.MAX)
    ms_step = float(t.item())
    value = work_units / (ms_step * 1e-3)

    # roofline of the dominant kernel (HBM; algorithmic bytes per launch / mean launch time)
    dom = max(stage_ms, key=lambda k: stage_ms[k])
    dom_bytes = unit_bytes[dom] * n
    achieved = dom_bytes / (stage_ms[dom] * 1e-3) / 1e9
    roofline = {"bound": "hbm", "kernel": dom, "achieved": achieved, "peak": hbm_peak, "unit": "GB/s",
                "frac": achieved / hbm_peak, "traffic": profiled_traffic(args.workload, n, dom), "peak_source": peak_src,
                "algorithmic_bytes_per_launch": dom_bytes}
    if cfg["kind"] == "cov":
        # every stage, and the pass as a whole, against the HBM roofline; K3's own bound is the
        # shared-memory atomic rate (tools/microbench/mb_dsmem: 1.355e12 returning adds/s on this pool's B200)
        per_stage = {k: {"algorithmic_GBps": unit_bytes[k] * n / (stage_ms[k] * 1e-3) / 1e9,
                         "frac_hbm": unit_bytes[k] * n / (stage_ms[k] * 1e-3) / 1e9 / hbm_peak}
                     for k in stage_ms if stage_ms[k] > 0 and unit_bytes[k] > 0}
        upd = n * m * (m + 1) / 2 / (stage_ms["covariance"] * 1e-3)
        per_stage["covariance"]["smem_atomic_updates_per_s"] = upd
        per_stage["covariance"]["frac_of_measured_atoms_peak"] = upd / 1.355e12  # mb_dsmem: returning atom.shared
        roofline["stages"] = per_stage
        roofline["pass_frac_hbm"] = (4 * p + 8 * m) * (n / (ms_step * 1e-3)) / 1e9 / hbm_peak

    out = {
        "metric": metric, "value": value, "unit": unit, "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": ms_step, "higher_is_better": True, "scaling": "weak", "vs_baseline": None,
        "dtype": args.compute if cfg["kind"] == "cov" else "f64",
        "data": "synthetic (seeded, device-generated; BASELINE.json generator shapes)",
        "config": {"workload": args.workload, "desc": cfg["desc"], "p": p, "m": m, "rows_per_gpu": n,
                   "sampler": args.sampler if cfg["kind"] == "cov" else "oracle",
                   "global_rows": total_samples, "parallelism": f"dp{world}",
                   "l2": "inputs larger than L2 (no flush needed)" if n * p * 4 > 126e6 else "inputs fit L2"},
        "stages_ms": stage_ms,
        "roofline": roofline,
        "gpu_launches": int(launches),
        "clocks": clk.summary(),
    }

    # secondary: the same pass with north_star's Philox sampler (not reference-identical
    # indices; pinned to oracle/sketch_oracle.c:orc_philox_indices), same shapes and timing
    if cfg["kind"] == "cov" and args.sampler == "oracle" and not args.no_philox:
        sampler = "philox"
        for _ in range(args.warmup):
            step(False)
        barrier()
        psums = [0.0] * len(stage_names)
        ksteps = max(1, min(args.steps, 5))
        p0 = torch.cuda.Event(enable_timing=True)
        p1 = torch.cuda.Event(enable_timing=True)
        p0.record()
        for _ in range(ksteps):
            step(True)
            torch.cuda.synchronize()
            for i in range(len(stage_names)):
                psums[i] += ev[i].elapsed_time(ev[i + 1])
        p1.record()
        barrier()
        pms = torch.tensor([p0.elapsed_time(p1) / ksteps], dtype=torch.float64, device=dev)
        if world > 1:
            tdist.all_reduce(pms, op=tdist.ReduceOp.MAX)
        out["philox_mode"] = {
            "value": n * world / (float(pms.item()) * 1e-3), "unit": unit, "ms_per_step": float(pms.item()),
            "stages_ms": {k: psums[i] / ksteps for i, k in enumerate(stage_names)},
            "gather_frac_hbm": unit_bytes["gather"] * n / (psums[1] / ksteps * 1e-3) / 1e9 / hbm_peak,
            "note": "skc_indices_philox + skc_sketch_given; uniform m-subsets, not the reference's subsets"}
        sampler = args.sampler

    # e2e through the public API with pinned host buffers
    if cfg["kind"] == "cov" and not args.no_e2e:
        n_e2e = min(n, 1 << 21)
        host = torch.empty((n_e2e, p), dtype=torch.float32, pin_memory=True)
        host.copy_(X[:n_e2e])
        src = skc.RowSource(host, chunk_cols=1 << 13)  # 32 MB chunks: copy k+1 hides chunk k's kernels

        def e2e_step():
            mom = skc.stream_moments(src, spec, plan, compute=args.compute, col0=col0)
            n_tot = sdist.combine_moments(mom.acc, mom.stats, mom.tri, mom.n)
            Cm = skc.covariance_from_moments(mom, p, m, n_tot)
            return Cm.cpu().numpy()

        e2e_step()
        barrier()
        w0 = time.perf_counter()
        for _ in range(max(1, min(args.steps, 3))):
            e2e_step()
        barrier()
        e_ms = (time.perf_counter() - w0) * 1e3 / max(1, min(args.steps, 3))
        te = torch.tensor([e_ms], dtype=torch.float64, device=dev)
        if world > 1:
            tdist.all_reduce(te, op=tdist.ReduceOp.MAX)
        e_ms = float(te.item())
        out["e2e"] = {"value": n_e2e * world / (e_ms * 1e-3), "unit": unit, "h2d_bytes_per_step": n_e2e * p * 4,
                      "d2h_bytes_per_step": p * p * 8, "rows_per_gpu": n_e2e,
                      "api": "stream_moments(RowSource(pinned host)) + covariance_from_moments: per-chunk sketch, "
                             "moments and covariance overlapped with the next chunk's H2D copy"}
        del host
    elif cfg["kind"] == "kmeans":
        out["e2e"] = {"value": None, "unit": unit, "note": "K-means e2e not measured in this mode"}

    # secondary: K-means C2 on the same box (rank 0 only, N=1)
    if cfg["kind"] == "cov" and not args.no_kmeans and world == 1 and args.workload == "c3":
        del X
        torch.cuda.empty_cache()
        c2 = WORKLOADS["c2"]
        X2 = gen_rows("c2", c2["n"], 0, dev, torch)
        spec2 = skc.PreconditionSpec.create("hadamard", c2["p"], sign_seed=derive_seed(SEED, 0xD5))
        plan2 = skc.SamplingPlan(derive_seed(SEED, 0x5A), spec2.p_pad, c2["m"])
        sk2 = skc.sketch_stream(skc.RowSource(X2), spec2, plan2, compute="f64")
        ops = skc.SketchKMeans(sk2)
        mu0 = ops.init_centers(np.random.default_rng(SEED).choice(c2["n"], c2["K"], replace=False))
        ops.lloyd(mu0, c2["iters"])
        torch.cuda.synchronize()
        reps = 5
        its, el = 0, 0.0
        for _ in range(reps):  # device time of each run (CUDA events inside the Lloyd loop)
            _, _, _, it_done, secs = ops.lloyd(mu0, c2["iters"])
            its += it_done
            el += secs
        out["kmeans_c2"] = {"metric": "K-means point-iters/s", "value": c2["n"] * its / el,
                            "iterations_per_run": its / reps, "ms_per_run": el * 1e3 / reps,
                            "note": "Lloyd loop on the HBM-resident f64 sketch, exact reference arithmetic"}
        if rank == 0 and not args.no_cpu:
            rows2 = X2[: 1 << 16].cpu().numpy()
            r, el2 = cpu_kmeans_rate(rows2, c2, os.cpu_count() or 1, min_seconds=5.0)
            out["kmeans_c2"]["cpu_baseline"] = {"value": r, "unit": "point-iters/s", "cores": os.cpu_count(),
                                                "kind": "port", "sample": "65536 C2 rows"}
        del X2, sk2, ops
        torch.cuda.empty_cache()
        if not args.no_c5:
            out["kmeans_c5"] = kmeans_secondary("c5", dev, torch, skc, hbm_peak)

    if rank == 0 and world == 1 and not args.no_cpu:
        sample_rows = 1 << 16
        Xs = gen_rows(args.workload, sample_rows, 0, dev, torch).cpu().numpy()
        nthreads = os.cpu_count() or 1
        if cfg["kind"] == "cov":
            rate, el = cpu_cov_rate(Xs, cfg, nthreads, min_seconds=10.0)
        else:
            rate, el = cpu_kmeans_rate(Xs, cfg, nthreads, min_seconds=10.0)
        out["cpu_baseline"] = {"value": rate, "unit": unit, "cores": nthreads, "kind": "port",
                               "sample": f"{sample_rows} rows of {args.workload}, repeated for {el:.1f}s"}

    if rank == 0:
        print(json.dumps(out), flush=True)
    if world > 1:
        tdist.destroy_process_group()


if __name__ == "__main__":
    main()
