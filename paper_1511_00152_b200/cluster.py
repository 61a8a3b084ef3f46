"""Sparsified K-means on a GPU sketch; the drop-in for cluster.py:28-404 (hot-path part).

Per Lloyd iteration on the device:
  K5 ``skc_kmeans_assign``    distances over each point's m sampled coordinates,
                              bit-exact fp64 (scipy CSR x dense axpy order)
     ``skc_pairwise_sum``     objective sum(d2min) in numpy's pairwise order
  K6 ``skc_kmeans_partials``  per-(j,k) sums and sampling counts, deterministic
     ``skc_kmeans_centers``   divide / keep previous / empty flags
     ``skc_kmeans_reseed``    empty clusters take the farthest point (cluster.py:212-215)
One small device-to-host read per iteration (changed-label count, objective, reseed
row) drives the stopping rule of cluster.py:235-236.
"""

from __future__ import annotations

import ctypes
import os
import time
from dataclasses import dataclass, field
from typing import Optional

import numpy as np
import torch

from . import _lib
from . import dist
from .errors import ParameterError
from .sketch import SparseSketch, as_source, device_row_chunks, plan_for, sketch_stream
from .transform import PreconditionSpec, unprecondition_columns

ORIGINAL = "original"
PRECONDITIONED = "preconditioned"
_TAG_RUN_SIGN, _TAG_RUN_SAMPLE = 0xD5, 0x5A  # cluster.py:362-363


@dataclass
class CenterSet:
    K: int
    centers: np.ndarray  # (p, K)
    domain: str = ORIGINAL


@dataclass
class Assignments:
    labels: np.ndarray  # (n,)


@dataclass
class CountDiagonal:
    """Per-cluster, per-coordinate sampling counts n_k^(j), shape (p, K); cluster.py:40-59"""

    counts: np.ndarray

    def cluster_sizes(self, m: int) -> np.ndarray:
        return self.counts.sum(axis=0) // m

    def hk_deviations(self, m: int) -> np.ndarray:
        p = self.counts.shape[0]
        n_k = self.counts.sum(axis=0) / m
        safe = np.where(n_k > 0, n_k, 1.0)
        dev = np.abs(p * self.counts / (m * safe)[None, :] - 1.0).max(axis=0)
        return np.where(n_k > 0, dev, np.nan)


@dataclass
class KMeansResult:
    assignments: Assignments
    centers: CenterSet
    objective: float
    diagnostics: dict = field(default_factory=dict)


def derive_seed(seed: int, tag: int) -> int:
    """_hash.py:33-35 (splitmix64 of seed ^ tag), evaluated on the host for the two run seeds."""
    z = (int(seed) ^ int(tag)) & 0xFFFFFFFFFFFFFFFF
    M = 0xFFFFFFFFFFFFFFFF
    z = ((z ^ (z >> 30)) * 0xBF58476D1CE4E5B9) & M
    z = ((z ^ (z >> 27)) * 0x94D049BB133111EB) & M
    return z ^ (z >> 31)


class SketchKMeans:
    """Device state of the sparsified Lloyd iteration on one sketch (the _SparseOps analogue)."""

    def __init__(self, sketch: SparseSketch):
        self.sketch = sketch
        self.n, self.m, self.p = sketch.n, sketch.m, sketch.p
        self.dev = sketch.indices.device
        self.idx = sketch.indices.contiguous()
        self.val = sketch.values.contiguous()
        self.vcode = _lib.dtype_code(self.val)
        self.col0 = int(getattr(sketch, "col0", 0))
        self._ws = {}

    def _workspace(self, key, nbytes):
        w = self._ws.get(key)
        if w is None or w.numel() < nbytes:
            w = _lib.workspace(nbytes, self.dev)
            self._ws[key] = w
        return w

    def _st(self):
        return _lib.stream_ptr(self.dev)

    def init_centers(self, chosen) -> torch.Tensor:
        """cluster.py:175-179"""
        ch = torch.as_tensor(np.asarray(chosen, dtype=np.int64), device=self.dev)
        K = int(ch.numel())
        mu = torch.empty((self.p, K), dtype=torch.float64, device=self.dev)
        with torch.cuda.device(self.dev):
            _lib.call("skc_kmeans_init", self.idx.data_ptr(), self.val.data_ptr(), self.vcode, self.n, self.m,
                      ch.data_ptr(), K, self.p, mu.data_ptr(), self._st())
        return mu

    def _use_tc(self, K: int) -> bool:
        # K5t (tensor-core filter) for tables beyond shared memory; SKC_ASSIGN_TC=0 disables it
        if os.environ.get("SKC_ASSIGN_TC", "1") == "0":
            return False
        L = _lib.lib()
        return self.p * K * 16 > 40 * 1024 and K > 16 and L.skc_kmeans_tc_supported(self.p, K, self.m) == 1

    def _tcprep(self) -> torch.Tensor:
        """Once per sketch: the compact bf16 entries and row norms of the tensor-core filter."""
        if "tcprep" not in self._ws:
            L = _lib.lib()
            prep = _lib.workspace(L.skc_kmeans_tc_prepare_workspace(self.n, self.m, self.p), self.dev)
            with torch.cuda.device(self.dev):
                _lib.call("skc_kmeans_tc_prepare", self.idx.data_ptr(), self.val.data_ptr(), self.vcode, self.n,
                          self.m, self.p, prep.data_ptr(), prep.numel(), self._st())
            self._ws["tcprep"] = prep
        return self._ws["tcprep"]

    def _csc(self) -> torch.Tensor:
        """Once per sketch: per-coordinate lists ascending in point index (skc_kmeans_build_csc)."""
        if "csc" not in self._ws:
            L = _lib.lib()
            csc = _lib.workspace(L.skc_kmeans_csc_workspace(self.n, self.m, self.p, self.vcode), self.dev)
            with torch.cuda.device(self.dev):
                _lib.call("skc_kmeans_build_csc", self.idx.data_ptr(), self.val.data_ptr(), self.vcode, self.n,
                          self.m, self.p, csc.data_ptr(), csc.numel(), self._st())
            self._ws["csc"] = csc
        return self._ws["csc"]

    def prepare(self, K: int) -> None:
        """Build the once-per-sketch structures the Lloyd iterations reuse (the transposed sketch,
        and for large centre tables the tensor-core entries), so they stay out of iteration timing."""
        self._csc()
        if self._use_tc(K):
            self._tcprep()

    def assign(self, mu: torch.Tensor, prev: Optional[torch.Tensor], labels: torch.Tensor, d2min: torch.Tensor,
               out: torch.Tensor, d2max: torch.Tensor) -> None:
        """cluster.py:181-187 (+ changed count vs prev, first argmax of d2min)"""
        K = mu.shape[1]
        L = _lib.lib()
        # the first assignment (prev is None) is from seeded or K-means++ centres, which are
        # sparse: nearly every point has near-ties there, and the fp32 filter (K5f) is the faster
        if prev is not None and self._use_tc(K):
            prep = self._tcprep()
            ws = self._workspace(("assign_tc", K), L.skc_kmeans_assign_tc_workspace(self.n, self.p, K))
            with torch.cuda.device(self.dev):
                _lib.call("skc_kmeans_assign_tc", self.idx.data_ptr(), self.val.data_ptr(), self.vcode, self.n,
                          self.m, mu.data_ptr(), self.p, K, _lib.ptr(prev), labels.data_ptr(), d2min.data_ptr(),
                          out.data_ptr(), d2max.data_ptr(), prep.data_ptr(), ws.data_ptr(), ws.numel(), self._st())
            return
        ws = self._workspace("assign", L.skc_kmeans_assign_workspace(self.n, self.p, K))
        with torch.cuda.device(self.dev):
            _lib.call("skc_kmeans_assign", self.idx.data_ptr(), self.val.data_ptr(), self.vcode, self.n, self.m,
                      mu.data_ptr(), self.p, K, _lib.ptr(prev), labels.data_ptr(), d2min.data_ptr(),
                      out.data_ptr(), d2max.data_ptr(), ws.data_ptr(), ws.numel(), self._st())

    def objective(self, d2min: torch.Tensor, out: torch.Tensor) -> None:
        L = _lib.lib()
        ws = self._workspace("pairwise", L.skc_pairwise_sum_workspace(self.n))
        with torch.cuda.device(self.dev):
            _lib.call("skc_pairwise_sum", d2min.data_ptr(), self.n, out.data_ptr(), ws.data_ptr(), ws.numel(),
                      self._st())

    def partials(self, labels: torch.Tensor, K: int):
        """cluster.py:189-208 partial sums: (sums, counts, sizes) on the device.

        Sums follow the reference's sequential order exactly, through the transposed sketch
        built on first use (``skc_kmeans_build_csc``)."""
        L = _lib.lib()
        csc = self._csc()
        seg = self._workspace(("seg", K), L.skc_kmeans_seg_workspace(self.n, self.m, self.p, K, self.vcode))
        sums = torch.empty((self.p, K), dtype=torch.float64, device=self.dev)
        counts = torch.empty((self.p, K), dtype=torch.int64, device=self.dev)
        sizes = torch.empty(K, dtype=torch.int64, device=self.dev)
        with torch.cuda.device(self.dev):
            _lib.call("skc_kmeans_partials_csc", csc.data_ptr(), self.vcode, self.n, self.m, self.p, labels.data_ptr(),
                      K, sums.data_ptr(), counts.data_ptr(), sizes.data_ptr(), seg.data_ptr(), seg.numel(),
                      self._st())
        return sums, counts, sizes

    def centers(self, sums, counts, sizes, mu_prev):
        """cluster.py:196-210 -> (mu, empty int32)"""
        K = mu_prev.shape[1]
        mu = torch.empty_like(mu_prev)
        empty = torch.empty(K, dtype=torch.int32, device=self.dev)
        with torch.cuda.device(self.dev):
            _lib.call("skc_kmeans_centers", sums.data_ptr(), counts.data_ptr(), sizes.data_ptr(), mu_prev.data_ptr(),
                      self.p, K, mu.data_ptr(), empty.data_ptr(), self._st())
        return mu, empty

    def reseed(self, mu, empty, idx_row: torch.Tensor, val_row: torch.Tensor) -> None:
        """cluster.py:212-215 for every empty cluster, with the farthest point's sketch row."""
        K = mu.shape[1]
        with torch.cuda.device(self.dev):
            _lib.call("skc_kmeans_reseed", idx_row.data_ptr(), val_row.data_ptr(), self.vcode, self.m,
                      empty.data_ptr(), self.p, K, mu.data_ptr(), self._st())

    def reseed_at(self, mu, empty, row: torch.Tensor) -> None:
        """reseed with the farthest point's row taken from device memory (row: int64[1])."""
        K = mu.shape[1]
        with torch.cuda.device(self.dev):
            _lib.call("skc_kmeans_reseed_at", self.idx.data_ptr(), self.val.data_ptr(), self.vcode, self.n, self.m,
                      row.data_ptr(), empty.data_ptr(), self.p, K, mu.data_ptr(), self._st())

    def update(self, labels: torch.Tensor, mu_prev: torch.Tensor, group=None):
        sums, counts, sizes = self.partials(labels, mu_prev.shape[1])
        if dist.world(group) > 1:
            for t in (sums, counts, sizes):
                dist.allreduce_(t, group=group)
        mu, empty = self.centers(sums, counts, sizes, mu_prev)
        return mu, counts, empty

    def lloyd(self, mu0: torch.Tensor, max_iter: int, group=None):
        return lloyd_loop(self, mu0, max_iter, group)


def lloyd_loop(ops, mu0: torch.Tensor, max_iter: int, group=None):
    """The _lloyd_iterate loop body from given centres; cluster.py:230-241.

    ``ops`` holds one shard (or all) of the sketch; with a process group of size > 1
    the reductions of dist.py make every rank follow the same trajectory.
    Returns (labels int32 on ops' device, mu, objective trajectory, iterations, seconds
    measured with CUDA events).
    """
    w = dist.world(group)
    if w == 1 and getattr(ops, "dev", torch.device("cpu")).type == "cuda" and hasattr(ops, "reseed_at"):
        if isinstance(ops, SketchKMeans) and os.environ.get("SKC_LLOYD", "graph") == "graph":
            return _lloyd_loop_graph(ops, mu0, max_iter)
        return _lloyd_loop_device(ops, mu0, max_iter)
    if w > 1:
        return _lloyd_loop_sharded(ops, mu0, max_iter, group)
    mu = mu0.clone()
    n, dev = ops.n, ops.dev
    lab = [torch.empty(n, dtype=torch.int32, device=dev) for _ in range(2)]
    d2min = torch.empty(n, dtype=torch.float64, device=dev)
    out = torch.zeros(2, dtype=torch.int64, device=dev)
    d2max = torch.zeros(1, dtype=torch.float64, device=dev)
    obj = torch.zeros(1, dtype=torch.float64, device=dev)
    stage = torch.empty(2, dtype=torch.float64, device=dev)
    traj, iters, prev = [], 0, None
    cur = lab[0]
    timed = dev.type == "cuda"
    if timed:
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        e0.record()
    for it in range(max_iter):
        cur = lab[it % 2]
        ops.assign(mu, prev, cur, d2min, out, d2max)
        ops.objective(d2min, obj)
        stage[0:1].copy_(out[0:1])  # changed (exact below 2^53)
        stage[1:2].copy_(obj)
        host = stage.cpu()  # the one device-to-host read of the iteration
        changed, objective = int(host[0]), float(host[1])
        traj.append(objective)
        iters += 1
        if prev is not None and changed == 0:
            break
        prev = cur
        mu, _, empty = ops.update(cur, mu, group)
        r = max(int(out[1]), 0)  # reseed point: first argmax of d2min (cluster.py:213)
        ops.reseed(mu, empty, ops.idx[r], ops.val[r])
    secs = 0.0
    if timed:
        e1.record()
        e1.synchronize()
        secs = e0.elapsed_time(e1) * 1e-3
    return cur, mu, traj, iters, secs


def _lloyd_loop_sharded(ops, mu0: torch.Tensor, max_iter: int, group=None):
    """cluster.py:230-241 over a sample-sharded sketch; every rank follows the same trajectory.

    Per iteration ONE SUM allreduce of the packed exchange (``skc_kmeans_pack_exchange``
    layout): [sums | counts | sizes | changed | objective | per rank (max d2min, global row of
    its first argmax)]. The partial sums are formed speculatively before the convergence test,
    as the single-GPU graph does; a converged iteration discards them. Only an iteration that
    empties a cluster adds one more allreduce, of the reseed row (SPEC.md:212, :352 ordered
    combine; the owner of the global first argmax is found from every rank's actual range).
    """
    w, me = dist.world(group), dist.rank(group)
    mu = mu0.clone()
    n, dev, p, m = ops.n, ops.dev, ops.p, ops.m
    K = int(mu.shape[1])
    pk = p * K
    ranges = dist.shard_ranges(int(ops.col0), n, dev, group)
    lab = [torch.empty(n, dtype=torch.int32, device=dev) for _ in range(2)]
    d2min = torch.empty(n, dtype=torch.float64, device=dev)
    out = torch.zeros(2, dtype=torch.int64, device=dev)
    d2max = torch.zeros(1, dtype=torch.float64, device=dev)
    obj = torch.zeros(1, dtype=torch.float64, device=dev)
    buf = torch.zeros(2 * pk + K + 2 + 2 * w, dtype=torch.float64, device=dev)
    on_gpu = dev.type == "cuda" and isinstance(ops, SketchKMeans)
    traj, iters, prev = [], 0, None
    cur = lab[0]
    timed = dev.type == "cuda"
    if timed:
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        e0.record()
    for it in range(max_iter):
        cur = lab[it % 2]
        ops.assign(mu, prev, cur, d2min, out, d2max)
        ops.objective(d2min, obj)
        sums, counts, sizes = ops.partials(cur, K)
        if on_gpu:
            with torch.cuda.device(dev):
                _lib.call("skc_kmeans_pack_exchange", sums.data_ptr(), counts.data_ptr(), sizes.data_ptr(),
                          out.data_ptr(), d2max.data_ptr(), obj.data_ptr(), p, K, me, w, int(ops.col0),
                          buf.data_ptr(), _lib.stream_ptr(dev))
        else:
            buf.zero_()
            buf[:pk] = sums.reshape(-1)
            buf[pk:2 * pk] = counts.reshape(-1).to(torch.float64)
            buf[2 * pk:2 * pk + K] = sizes.to(torch.float64)
            buf[2 * pk + K] = out[0].to(torch.float64)
            buf[2 * pk + K + 1] = obj[0]
            slot = 2 * pk + K + 2 + 2 * me
            buf[slot] = d2max[0]
            buf[slot + 1] = float(int(ops.col0) + int(out[1])) if int(out[1]) >= 0 else -1.0
        dist.allreduce_(buf, group=group)  # the one collective of the iteration
        host = buf[2 * pk:].cpu()  # the one device-to-host read: sizes, changed, objective, slots
        changed, objective = int(host[K]), float(host[K + 1])
        traj.append(objective)
        iters += 1
        if prev is not None and changed == 0:
            break
        prev = cur
        sums_g = buf[:pk].view(p, K)
        counts_g = buf[pk:2 * pk].view(p, K).to(torch.int64)
        sizes_g = buf[2 * pk:2 * pk + K].to(torch.int64)
        mu, empty = ops.centers(sums_g, counts_g, sizes_g, mu)
        if bool((host[:K] == 0).any()):
            # reseed point: global first argmax of d2min (cluster.py:213, np.argmax semantics)
            slots = host[K + 2:].view(w, 2)
            vmax = float(slots[:, 0].max())
            g = min(int(slots[q, 1]) for q in range(w) if float(slots[q, 0]) == vmax and slots[q, 1] >= 0)
            owner = next(q for q, (c0, nq) in enumerate(ranges) if c0 <= g < c0 + nq)
            row = torch.zeros(2 * m, dtype=torch.float64, device=dev)
            if me == owner:
                row[:m] = ops.idx[g - ranges[me][0]].to(torch.float64)
                row[m:] = ops.val[g - ranges[me][0]].to(torch.float64)
            dist.allreduce_(row, group=group)
            ops.reseed(mu, empty, row[:m].to(torch.int32), row[m:].to(ops.val.dtype))
    secs = 0.0
    if timed:
        e1.record()
        e1.synchronize()
        secs = e0.elapsed_time(e1) * 1e-3
    return cur, mu, traj, iters, secs


def _lloyd_loop_graph(ops: "SketchKMeans", mu0: torch.Tensor, max_iter: int):
    """Single-GPU Lloyd loop as one device-resident CUDA graph (``skc_kmeans_lloyd``).

    The iterations, including the convergence test of cluster.py:235-236, run inside a graph
    with a conditional WHILE node: no host round trip per iteration. The host reads the
    trajectory and the iteration count once, after the loop. Same kernels, same arithmetic
    and the same trajectory as lloyd_loop (cluster.py:230-241).
    """
    L = _lib.lib()
    n, m, p, K = ops.n, ops.m, ops.p, int(mu0.shape[1])
    max_iter = int(max_iter)
    use_tc = ops._use_tc(K)
    csc = ops._csc()
    prep = ops._tcprep() if use_tc else None
    ws = ops._workspace(("lloyd_ws", K, use_tc), L.skc_kmeans_lloyd_workspace(n, m, p, K, ops.vcode, int(use_tc)))
    key = ("lloyd_bufs", K, max_iter)
    bufs = ops._ws.get(key)
    if bufs is None:
        bufs = dict(mu0=torch.empty((p, K), dtype=torch.float64, device=ops.dev),
                    mu=torch.empty((p, K), dtype=torch.float64, device=ops.dev),
                    labels=torch.empty(n, dtype=torch.int32, device=ops.dev),
                    res=torch.zeros(max_iter + 1, dtype=torch.float64, device=ops.dev),
                    host=torch.empty(max_iter + 1, dtype=torch.float64, pin_memory=True))
        ops._ws[key] = bufs
    res = bufs["res"]
    traj_d, iters_d = res[:max_iter], res[max_iter:].view(torch.int32)
    e0 = torch.cuda.Event(enable_timing=True)
    e1 = torch.cuda.Event(enable_timing=True)
    with torch.cuda.device(ops.dev):
        e0.record()
        bufs["mu0"].copy_(mu0)
        _lib.call("skc_kmeans_lloyd", ops.idx.data_ptr(), ops.val.data_ptr(), ops.vcode, n, m, p, K,
                  bufs["mu0"].data_ptr(), max_iter, csc.data_ptr(), _lib.ptr(prep), ws.data_ptr(), ws.numel(),
                  bufs["labels"].data_ptr(), bufs["mu"].data_ptr(), traj_d.data_ptr(), iters_d.data_ptr(),
                  ops._st())
        bufs["host"].copy_(res, non_blocking=True)  # the loop's one device-to-host read
        e1.record()
        e1.synchronize()
    host = bufs["host"]
    iters = int(host[max_iter:].view(torch.int32)[0])
    traj = [float(v) for v in host[:iters]]
    pro, body = _c_int32(), _c_int32()
    L.skc_kmeans_lloyd_graph_kernels(ctypes.byref(pro), ctypes.byref(body))
    L.skc_count_launches(pro.value + (iters - 1) * body.value)
    return bufs["labels"].clone(), bufs["mu"].clone(), traj, iters, e0.elapsed_time(e1) * 1e-3


def _c_int32():
    return ctypes.c_int32(0)


def _lloyd_loop_device(ops, mu0: torch.Tensor, max_iter: int):
    """Single-GPU Lloyd loop with one host read per iteration, overlapped with the next step.

    Each iteration enqueues assign + objective, a 32-byte device-to-host copy of
    (changed, argmax row, objective, max d2), and then, speculatively, the update and the
    reseed (which takes the argmax row from device memory). The host waits only for the
    copy; on convergence the speculative centres are discarded. The arithmetic and the
    trajectory equal lloyd_loop's (cluster.py:230-241).
    """
    n, dev = ops.n, ops.dev
    mu = mu0.clone()
    lab = [torch.empty(n, dtype=torch.int32, device=dev) for _ in range(2)]
    d2min = torch.empty(n, dtype=torch.float64, device=dev)
    raw = torch.zeros(32, dtype=torch.uint8, device=dev)
    out, obj, d2max = raw[0:16].view(torch.int64), raw[16:24].view(torch.float64), raw[24:32].view(torch.float64)
    host = torch.empty(32, dtype=torch.uint8, pin_memory=True)
    h_out, h_obj = host[0:16].view(torch.int64), host[16:24].view(torch.float64)
    ready = torch.cuda.Event()
    e0 = torch.cuda.Event(enable_timing=True)
    e1 = torch.cuda.Event(enable_timing=True)
    traj, iters, prev = [], 0, None
    cur = lab[0]
    e0.record()
    for it in range(max_iter):
        cur = lab[it % 2]
        ops.assign(mu, prev, cur, d2min, out, d2max)
        ops.objective(d2min, obj)
        host.copy_(raw, non_blocking=True)
        ready.record()
        mu_next, _, empty = ops.update(cur, mu)
        ops.reseed_at(mu_next, empty, out[1:2])
        ready.synchronize()
        changed, objective = int(h_out[0]), float(h_obj[0])
        traj.append(objective)
        iters += 1
        if prev is not None and changed == 0:
            break
        prev = cur
        mu = mu_next
    e1.record()
    e1.synchronize()
    return cur, mu, traj, iters, e0.elapsed_time(e1) * 1e-3


def _labels_to_device(labels, dev) -> torch.Tensor:
    if isinstance(labels, torch.Tensor):
        return labels.to(device=dev, dtype=torch.int32).contiguous()
    return torch.as_tensor(np.asarray(labels, dtype=np.int64), device=dev).to(torch.int32)


def sparsified_assign(sketch: SparseSketch, i: int, mu_prime: CenterSet) -> int:
    """Nearest centre for one column over its m sampled coordinates; cluster.py:306-311.

    ``skc_kmeans_assign_one`` evaluates the reference's own expression for this call,
    ((val[:, None] - mu[idx]) ** 2).sum(axis=0), in its order (a sequential sum over the m
    coordinates), so near-ties resolve as the reference does; ties go to the lowest index.
    """
    dev = sketch.indices.device
    mu = torch.as_tensor(np.asarray(mu_prime.centers, dtype=np.float64), device=dev).contiguous()
    K = int(mu.shape[1])
    idx = sketch.indices[i].contiguous()
    val = sketch.values[i].contiguous()
    lab = torch.empty(1, dtype=torch.int32, device=dev)
    with torch.cuda.device(dev):
        _lib.call("skc_kmeans_assign_one", idx.data_ptr(), val.data_ptr(), _lib.dtype_code(val), sketch.m,
                  mu.data_ptr(), sketch.p, K, lab.data_ptr(), None, _lib.stream_ptr(dev))
    return int(lab.item())


def sparsified_update_centers(sketch: SparseSketch, assignments: Assignments, K: int = None,
                              prev_centers: CenterSet = None):
    """Entry-wise sample means per cluster + sampling counts; cluster.py:314-339"""
    labels = np.asarray(assignments.labels.cpu() if isinstance(assignments.labels, torch.Tensor)
                        else assignments.labels, dtype=np.int64)
    if K is None:
        K = int(labels.max()) + 1
    if labels.size and (labels.min() < 0 or labels.max() >= K):
        raise ParameterError("labels must lie in [0, K)")
    ops = SketchKMeans(sketch)
    mu_prev = (torch.as_tensor(np.asarray(prev_centers.centers, dtype=np.float64), device=ops.dev).contiguous()
               if prev_centers is not None else torch.zeros((sketch.p, K), dtype=torch.float64, device=ops.dev))
    mu, counts, _ = ops.update(_labels_to_device(labels, ops.dev), mu_prev)
    return (CenterSet(K=K, centers=mu.cpu().numpy(), domain=PRECONDITIONED),
            CountDiagonal(counts=counts.cpu().numpy()))


def _initial_centers(ops: SketchKMeans, K: int, init, restart: int, seed: int) -> torch.Tensor:
    """Point indices are global (col0-relative shards under torch.distributed)."""
    if init is None:
        from .kmeanspp import kmeanspp_select

        chosen = kmeanspp_select(ops, K, seed, restart)
        return dist.init_centers_global(ops, chosen)
    if isinstance(init, CenterSet):
        return torch.as_tensor(np.asarray(init.centers, dtype=np.float64), device=ops.dev).contiguous()
    arr = np.asarray(init)
    if arr.ndim == 1:  # K chosen point indices (init_centers semantics)
        if arr.shape[0] != K:
            raise ParameterError(f"init lists {arr.shape[0]} points, K={K}")
        return dist.init_centers_global(ops, arr.astype(np.int64))
    if arr.ndim == 2 and arr.shape == (ops.p, K):
        return torch.as_tensor(arr.astype(np.float64), device=ops.dev).contiguous()
    raise ParameterError("init must be K point indices or a (p_pad, K) centre matrix")


def _sparsified_on_sketch(sketch: SparseSketch, K: int, max_iter: int = 100, n_init: int = 20, seed: int = 0,
                          init=None) -> KMeansResult:
    """cluster.py:375-404. ``init`` (K point indices or centres) replaces K-means++ and
    runs a single restart. On a sharded sketch (world > 1) every rank follows the same
    restarts and trajectory; the labels are this rank's shard, the rest is global."""
    ops = SketchKMeans(sketch)
    restarts = 1 if init is not None else int(n_init)
    best, iter_seconds, iters_total = None, 0.0, 0
    for r in range(restarts):
        mu0 = _initial_centers(ops, K, init, r, seed)
        labels, mu, traj, iters, secs = ops.lloyd(mu0, max_iter)
        iter_seconds += secs
        iters_total += iters
        if best is None or traj[-1] < best[2][-1]:
            best = (labels.clone(), mu, traj, iters)
    labels, mu, traj, iters = best
    _, counts, _ = ops.update(labels, mu)  # sums the shards' counts under world > 1
    spec = sketch.spec
    back = unprecondition_columns(mu, spec)[: spec.p]
    mu_h = mu.cpu().numpy()
    return KMeansResult(
        assignments=Assignments(labels=labels.cpu().numpy().astype(np.int64)),
        centers=CenterSet(K=K, centers=back.cpu().numpy(), domain=ORIGINAL),
        objective=traj[-1],
        diagnostics={
            "iterations": iters,
            "iterations_total": iters_total,
            "objective_curve": traj,
            "iter_seconds": iter_seconds,
            "restarts": restarts,
            "m": sketch.m,
            "p_pad": sketch.p,
            "centers_preconditioned": CenterSet(K=K, centers=mu_h, domain=PRECONDITIONED),
            "count_diagonal": CountDiagonal(counts=counts.cpu().numpy()),
        },
    )


def sparsified_kmeans(source, K: int, gamma: float, max_iter: int = 100, n_init: int = 20, seed: int = 0,
                      kind: str = "hadamard", chunk_cols: int = 8192, *, init=None, compute: str = "f64",
                      device=None, col0: Optional[int] = None) -> KMeansResult:
    """One-pass sparsified K-means; cluster.py:342-372.

    Under torch.distributed (world > 1) ``source`` is this rank's shard of the columns, at
    global offset ``col0`` (default: shards concatenated in rank order). ``init`` point
    indices are global; the returned labels are the shard's, centres and objective global."""
    source = as_source(source, chunk_cols=chunk_cols)
    c0, n_total = dist.shard_offset(source.n)
    if col0 is not None:
        c0 = int(col0)
    if K > n_total:
        raise ParameterError(f"K={K} exceeds number of points n={n_total}")
    spec = PreconditionSpec.create(kind, source.p, sign_seed=derive_seed(seed, _TAG_RUN_SIGN))
    plan = plan_for(spec, gamma, master_seed=derive_seed(seed, _TAG_RUN_SAMPLE))
    t0 = time.perf_counter()
    sketch = sketch_stream(source, spec, plan, compute=compute, device=device, col0=c0)
    torch.cuda.synchronize(sketch.indices.device)
    sketch_seconds = time.perf_counter() - t0
    result = _sparsified_on_sketch(sketch, K, max_iter=max_iter, n_init=n_init, seed=seed, init=init)
    result.diagnostics.update(sketch_seconds=sketch_seconds, passes=getattr(source, "passes", None))
    return result


def sparsified_kmeans_two_pass(source, K: int, gamma: float, max_iter: int = 100, n_init: int = 20, seed: int = 0,
                               kind: str = "hadamard", chunk_cols: int = 8192, *, compute: str = "f64",
                               device=None, col0: Optional[int] = None) -> KMeansResult:
    """Sparsified K-means plus one pass over the raw rows; cluster.py:407-456.

    The second pass runs on the GPU as the raw chunks stream in (pinned copies overlapped
    with the kernels): ``skc_dense_assign`` re-assigns every point to its nearest first-pass
    centre (first argmin of (|x|^2 - 2 <x, mu>) + |mu|^2, clipped objective) and
    ``skc_dense_sums`` accumulates the exact original-domain means of the first-pass
    clusters. Nothing further is iterated. Each chunk's objective is a numpy-order pairwise
    sum, and the chunk sums add in chunk order, as the reference does. Sharded (world > 1):
    each rank passes its shard as in ``sparsified_kmeans``; the cluster sums and counts are
    allreduced and the chunk objectives add in rank order.
    """
    source = as_source(source, chunk_cols=chunk_cols)
    first = sparsified_kmeans(source, K, gamma, max_iter=max_iter, n_init=n_init, seed=seed, kind=kind,
                              chunk_cols=chunk_cols, compute=compute, device=device, col0=col0)
    dev = torch.device(device) if device is not None else torch.device("cuda", torch.cuda.current_device())
    mu_hat = np.asarray(first.centers.centers, dtype=np.float64)  # (p, K)
    p, n = source.p, source.n
    mu_rows = torch.as_tensor(np.ascontiguousarray(mu_hat.T), device=dev)  # (K, p)
    lab1 = torch.as_tensor(np.asarray(first.assignments.labels, dtype=np.int32), device=dev)
    labels2 = torch.empty(n, dtype=torch.int32, device=dev)
    d2min = torch.empty(n, dtype=torch.float64, device=dev)
    sums = torch.zeros((K, p), dtype=torch.float64, device=dev)
    counts = torch.zeros(K, dtype=torch.int64, device=dev)
    L = _lib.lib()
    aws = _lib.workspace(L.skc_dense_assign_workspace(p, K), dev)
    row_iter = source.row_chunks() if hasattr(source, "row_chunks") else (ch.T for ch in source.chunks())
    chunk_obj, spans = [], []
    j0 = 0
    with torch.cuda.device(dev):
        st = _lib.stream_ptr(dev)
        for rows in device_row_chunks(row_iter, dev):
            if rows.ndim != 2 or rows.shape[1] != p:
                raise ParameterError(f"bad chunk at column offset {j0}: expected ({p}, c)")
            if rows.stride(1) != 1:
                rows = rows.contiguous()
            c = rows.shape[0]
            if j0 + c > n:
                raise ParameterError(f"source yielded more than {n} columns")
            xc = _lib.dtype_code(rows)
            _lib.call("skc_dense_assign", rows.data_ptr(), xc, rows.stride(0), c, p, mu_rows.data_ptr(), K,
                      aws.data_ptr(), labels2[j0:].data_ptr(), d2min[j0:].data_ptr(), st)
            ws = _lib.workspace(L.skc_dense_sums_workspace(c, p, K), dev)
            _lib.call("skc_dense_sums", rows.data_ptr(), xc, rows.stride(0), c, p, lab1[j0:].data_ptr(), K,
                      sums.data_ptr(), counts.data_ptr(), ws.data_ptr(), st)
            spans.append((j0, c))
            j0 += c
        if j0 != n:
            raise ParameterError(f"source yielded {j0} columns, expected {n}")
        obj_dev = torch.zeros(max(len(spans), 1), dtype=torch.float64, device=dev)
        pw = _lib.workspace(L.skc_pairwise_sum_workspace(max((c for _, c in spans), default=1)), dev)
        for t, (a, c) in enumerate(spans):
            _lib.call("skc_pairwise_sum", d2min[a:].data_ptr(), c, obj_dev[t:].data_ptr(), pw.data_ptr(), pw.numel(), st)
        dist.allreduce_(sums)  # sharded (world > 1): every rank's first-pass cluster sums
        dist.allreduce_(counts)
    obj = dist.ordered_sum(obj_dev.cpu().numpy()[: len(spans)].tolist())  # chunk order, then rank order
    cnt = counts.cpu().numpy()
    mu2 = sums.cpu().numpy().T.copy()  # (p, K)
    nz = cnt > 0
    mu2[:, nz] = mu2[:, nz] / cnt[nz].astype(np.float64)[None, :]
    mu2[:, ~nz] = mu_hat[:, ~nz]
    diagnostics = dict(first.diagnostics)
    diagnostics.update(passes=getattr(source, "passes", None), first_pass_objective=first.objective)
    return KMeansResult(
        assignments=Assignments(labels=labels2.cpu().numpy().astype(np.int64)),
        centers=CenterSet(K=K, centers=mu2, domain=ORIGINAL),
        objective=obj,
        diagnostics=diagnostics,
    )
