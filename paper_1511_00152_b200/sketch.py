"""Single-pass precondition + sparsify on the GPU; the drop-in for sketch.py:1-223.

``sketch_stream`` is the fused operator K1. For every column it zero-pads, applies
D, runs the normalised WHT, keeps the m coordinates with the smallest splitmix64 keys,
and writes compact (index, value) rows. All of this is one kernel launch per chunk
(``skc_sketch``). Column i uses the GLOBAL column index, so any chunking, sharding or
launch order gives identical bytes (sketch.py:196-201).

Layout: the GPU works on sample-major rows. A (p, n) input block is read as its n
columns. Fortran-ordered arrays and (n, p) row sources are consumed without a copy.
Outputs live on the device: ``indices`` (n, m) int32 and ``values`` (n, m) fp64 or fp32.
"""

from __future__ import annotations

from dataclasses import dataclass
from typing import Iterator, Optional

import numpy as np
import torch

from . import _lib
from .errors import DimensionError, ParameterError
from .transform import PreconditionSpec, as_device, default_device, u64

DEFAULT_CHUNK_COLS = 8192
COMPUTE = {"f64": _lib.F64, "f32": _lib.F32}


SAMPLERS = ("oracle", "philox")


@dataclass(frozen=True)
class SamplingPlan:
    """Master seed plus (p, m); sketch.py:23-56. Indices are drawn on the GPU.

    ``sampler="oracle"`` (default) is the reference's keyed-hash rule, bit-exact.
    ``sampler="philox"`` is north_star's counter-based alternative: Floyd's algorithm on a
    Philox4x32-10 stream (``skc_indices_philox``). It draws from the same distribution
    (uniform m-subsets), but not the reference's subsets. It is much cheaper on the GPU and
    is pinned bit for bit against ``oracle/sketch_oracle.c:orc_philox_indices``.
    """

    master_seed: int
    p: int
    m: int
    sampler: str = "oracle"

    def __post_init__(self):
        if not 1 <= self.m <= self.p:
            raise ParameterError(f"need 1 <= m <= p, got m={self.m}, p={self.p}")
        if self.sampler not in SAMPLERS:
            raise ParameterError(f"sampler must be one of {SAMPLERS}, got {self.sampler!r}")

    @property
    def gamma(self) -> float:
        return self.m / self.p

    def indices(self, i: int) -> np.ndarray:
        """Sorted sampled coordinates of column i, shape (m,) uint32."""
        return self.indices_block(i, i + 1)[0]

    def device_indices(self, i0: int, i1: int, device=None) -> torch.Tensor:
        c = int(i1) - int(i0)
        out = torch.empty((max(c, 0), self.m), dtype=torch.int32, device=device or default_device())
        if c > 0:
            with torch.cuda.device(out.device):
                _lib.call("skc_indices" if self.sampler == "oracle" else "skc_indices_philox", u64(self.master_seed),
                          int(i0), c, self.p, self.m, out.data_ptr(), _lib.stream_ptr(out.device))
        return out

    def indices_block(self, i0: int, i1: int) -> np.ndarray:
        """Sampled coordinates for columns i0..i1-1, shape (i1-i0, m) uint32; sketch.py:48-56"""
        return self.device_indices(i0, i1).cpu().numpy().astype(np.uint32)


def sample_indices(plan: SamplingPlan, i: int) -> np.ndarray:
    """sketch.py:59-61"""
    return plan.indices(i)


@dataclass
class SparseSketch:
    """Per-column (index, value) pairs, exactly m per column; sketch.py:64-113.

    ``indices`` (n, m) and ``values`` (n, m) are CUDA tensors (int32 / fp64 or fp32).
    Row i is column i of the sketch. ``plan`` is None for hand-built sketches.
    """

    spec: PreconditionSpec
    n: int
    indices: torch.Tensor
    values: torch.Tensor
    plan: Optional[SamplingPlan] = None
    col0: int = 0

    @property
    def m(self) -> int:
        return int(self.indices.shape[1])

    @property
    def p(self) -> int:
        return self.spec.p_pad

    @classmethod
    def from_host(cls, spec, n, indices, values, plan=None, device=None, values_dtype=torch.float64):
        """Hand-built sketch (test_estimators.py:22-29 style) moved to the device."""
        device = device or default_device()
        idx = torch.as_tensor(np.asarray(indices).astype(np.int64)).to(device=device, dtype=torch.int32)
        val = torch.as_tensor(np.asarray(values, dtype=np.float64)).to(device=device, dtype=values_dtype)
        idx = idx.reshape(int(n), -1) if idx.numel() else idx.reshape(int(n), idx.shape[-1] if idx.ndim == 2 else 0)
        val = val.reshape(idx.shape)
        return cls(spec=spec, n=int(n), indices=idx.contiguous(), values=val.contiguous(), plan=plan)

    def host_indices(self) -> np.ndarray:
        return self.indices.cpu().numpy().astype(np.uint32)

    def host_values(self) -> np.ndarray:
        return self.values.cpu().numpy().astype(np.float64)

    def column(self, i: int):
        return self.host_indices()[i], self.host_values()[i]

    def to_csc(self):
        """(p, n) scipy CSC with explicit zeros kept, on the host; sketch.py:91-98"""
        import scipy.sparse as sp

        n, m = self.n, self.m
        indptr = np.arange(0, (n + 1) * m, m, dtype=np.int64)
        return sp.csc_matrix((self.host_values().ravel(), self.host_indices().ravel().astype(np.int64), indptr),
                             shape=(self.p, n))

    def pattern_csc(self):
        import scipy.sparse as sp

        n, m = self.n, self.m
        indptr = np.arange(0, (n + 1) * m, m, dtype=np.int64)
        return sp.csc_matrix((np.ones(n * m), self.host_indices().ravel().astype(np.int64), indptr), shape=(self.p, n))

    def densify(self) -> np.ndarray:
        """Dense (p, n) with unsampled coordinates zero; sketch.py:109-113 (scatter on the GPU)."""
        D = torch.zeros((self.n, self.p), dtype=torch.float64, device=self.indices.device)
        if self.n:
            D.scatter_(1, self.indices.long(), self.values.to(torch.float64))
        return D.T.cpu().numpy()


class ArraySource:
    """In-memory column source with chunking and a pass counter; sketch.py:143-167.

    ``X`` is a (p, n) matrix: numpy, or a torch tensor on the host or a CUDA device.
    """

    def __init__(self, X, chunk_cols: int = DEFAULT_CHUNK_COLS):
        if isinstance(X, torch.Tensor):
            if X.ndim != 2:
                raise DimensionError("expected a (p, n) matrix")
            if X.dtype not in (torch.float32, torch.float64):
                X = X.to(torch.float64)
        else:
            X = np.asarray(X)
            if X.ndim != 2:
                raise DimensionError("expected a (p, n) matrix")
            if X.dtype not in (np.float32, np.float64):
                X = X.astype(np.float64)
        if chunk_cols < 1:
            raise ParameterError("chunk_cols must be >= 1")
        self.X = X
        self.chunk_cols = int(chunk_cols)
        self.passes = 0

    @property
    def p(self) -> int:
        return int(self.X.shape[0])

    @property
    def n(self) -> int:
        return int(self.X.shape[1])

    def chunks(self) -> Iterator:
        self.passes += 1
        for j0 in range(0, self.n, self.chunk_cols):
            yield self.X[:, j0 : j0 + self.chunk_cols]

    def row_chunks(self) -> Iterator:
        """Sample-major (c, p) chunks. Zero-copy for Fortran-ordered / device data. One pass."""
        self.passes += 1
        if isinstance(self.X, torch.Tensor) and self.X.is_cuda:
            yield self.X.T  # one launch: the output does not depend on chunking
            return
        for j0 in range(0, self.n, self.chunk_cols):
            yield self.X[:, j0 : j0 + self.chunk_cols].T


class RowSource:
    """Sample-major source: ``rows`` is (n, p), row i = sample i (the GPU-native layout).

    Host rows are copied to the device chunk by chunk. CUDA rows are consumed in one
    launch.
    """

    def __init__(self, rows, chunk_cols: int = 1 << 16):
        if rows.ndim != 2:
            raise DimensionError("expected an (n, p) row matrix")
        self.rows = rows
        self.chunk_cols = int(chunk_cols)
        self.passes = 0

    @property
    def p(self) -> int:
        return int(self.rows.shape[1])

    @property
    def n(self) -> int:
        return int(self.rows.shape[0])

    def chunks(self):
        self.passes += 1
        for j0 in range(0, self.n, self.chunk_cols):
            yield self.rows[j0 : j0 + self.chunk_cols].T

    def row_chunks(self):
        self.passes += 1
        if isinstance(self.rows, torch.Tensor) and self.rows.is_cuda:
            yield self.rows
            return
        for j0 in range(0, self.n, self.chunk_cols):
            yield self.rows[j0 : j0 + self.chunk_cols]


def as_source(data, chunk_cols: int = DEFAULT_CHUNK_COLS):
    """Pass sources through unchanged; wrap raw matrices; sketch.py:170-174"""
    if hasattr(data, "chunks") and hasattr(data, "p") and hasattr(data, "n"):
        return data
    return ArraySource(data, chunk_cols=chunk_cols)


def plan_for(spec: PreconditionSpec, gamma: float, master_seed: int, sampler: str = "oracle") -> SamplingPlan:
    """Keep round(gamma * p_pad) entries per column; sketch.py:177-184"""
    if not 0 < gamma <= 1:
        raise ParameterError(f"gamma must be in (0, 1], got {gamma}")
    m = int(round(gamma * spec.p_pad))
    if m < 1:
        raise ParameterError(f"gamma={gamma} keeps no entries at p_pad={spec.p_pad}")
    return SamplingPlan(master_seed=int(master_seed), p=spec.p_pad, m=m, sampler=sampler)


def _launch_rows(rows: torch.Tensor, spec: PreconditionSpec, plan: SamplingPlan, col0: int, compute: int,
                 idx_out: torch.Tensor, val_out: torch.Tensor) -> None:
    """One skc_sketch launch over CUDA rows (c, p) -> idx_out/val_out (c, m) views."""
    if rows.stride(1) != 1:
        rows = rows.contiguous()
    c = rows.shape[0]
    if c == 0:
        return
    with torch.cuda.device(rows.device):
        st = _lib.stream_ptr(rows.device)
        if plan.sampler == "philox":
            _lib.call("skc_indices_philox", u64(plan.master_seed), int(col0), c, plan.p, plan.m, idx_out.data_ptr(), st)
            sketch_given_rows(rows, spec, plan.m, compute, idx_out, val_out)
            return
        _lib.call("skc_sketch", rows.data_ptr(), _lib.dtype_code(rows), rows.stride(0), c, spec.p, spec.p_pad,
                  spec.gpu_kind(), u64(spec.sign_seed), u64(plan.master_seed), int(col0), plan.m, compute,
                  idx_out.data_ptr(), val_out.data_ptr(), _lib.dtype_code(val_out), st)


def sketch_given_rows(rows: torch.Tensor, spec: PreconditionSpec, m: int, compute: int, idx_in: torch.Tensor,
                      val_out: torch.Tensor) -> None:
    """Values of CUDA rows (c, p) at supplied sorted indices (c, m) int32 (``skc_sketch_given``):
    oracle mode with reference-supplied indices, or the Philox sampler's."""
    if rows.stride(1) != 1:
        rows = rows.contiguous()
    c = rows.shape[0]
    if c == 0:
        return
    if tuple(idx_in.shape) != (c, m) or idx_in.dtype != torch.int32 or not idx_in.is_contiguous():
        raise DimensionError(f"indices must be contiguous int32 ({c}, {m})")
    with torch.cuda.device(rows.device):
        _lib.call("skc_sketch_given", rows.data_ptr(), _lib.dtype_code(rows), rows.stride(0), c, spec.p, spec.p_pad,
                  spec.gpu_kind(), u64(spec.sign_seed), m, compute, idx_in.data_ptr(), val_out.data_ptr(),
                  _lib.dtype_code(val_out), _lib.stream_ptr(rows.device))


def device_row_chunks(row_iter, device) -> Iterator[torch.Tensor]:
    """CUDA (c, p) row chunks from host or device chunks, copying ahead of the consumer.

    Host chunks (numpy or torch, any strides) go through two pinned staging buffers and a
    copy stream: chunk k+1's host-to-device copy runs while the caller's kernels consume
    chunk k on the current stream. Pinned contiguous torch chunks are copied directly.
    CUDA chunks pass through.
    """
    device = torch.device(device)
    copy_stream = None
    ring = [None, None]
    done = [None, None]
    for k, chunk in enumerate(row_iter):
        if isinstance(chunk, torch.Tensor) and chunk.is_cuda:
            yield chunk
            continue
        t = chunk if isinstance(chunk, torch.Tensor) else torch.from_numpy(np.asarray(chunk))
        if t.ndim != 2:
            raise DimensionError(f"bad chunk: expected a 2-D block, got shape {tuple(t.shape)}")
        if t.dtype not in (torch.float32, torch.float64):
            t = t.to(torch.float64)
        if copy_stream is None:
            copy_stream = torch.cuda.Stream(device)
        slot = k & 1
        if t.is_pinned() and t.is_contiguous():
            src = t
        else:
            if done[slot] is not None:
                done[slot].synchronize()  # the previous copy out of this staging buffer finished
            need = t.numel()
            buf = ring[slot]
            if buf is None or buf.dtype != t.dtype or buf.numel() < need:
                buf = ring[slot] = torch.empty(max(need, 1), dtype=t.dtype, pin_memory=True)
            src = buf[:need].view(t.shape)
            src.copy_(t)
        compute = torch.cuda.current_stream(device)
        with torch.cuda.stream(copy_stream):
            dev = torch.empty(t.shape, dtype=t.dtype, device=device)
            dev.copy_(src, non_blocking=True)
            ev = torch.cuda.Event()
            ev.record(copy_stream)
        done[slot] = ev
        compute.wait_event(ev)
        dev.record_stream(compute)
        yield dev


def sketch_stream(source, spec: PreconditionSpec, plan: SamplingPlan, *, compute: str = "f64",
                  values_dtype: Optional[torch.dtype] = None, device=None, col0: int = 0,
                  indices=None) -> SparseSketch:
    """Precondition and sample every column of ``source`` in one pass; sketch.py:196-223.

    compute="f64" reproduces the reference values bit for bit. compute="f32" is the
    fast path. Indices are bit-exact in both. ``col0`` offsets the global column index,
    for a shard of a larger matrix. ``indices`` (n, m), each row strictly increasing,
    replaces sampling: the values are taken at those coordinates (oracle mode with
    reference-supplied indices).
    """
    source = as_source(source)
    if source.p != spec.p:
        raise DimensionError(f"source has p={source.p}, spec expects {spec.p}")
    if plan.p != spec.p_pad:
        raise DimensionError("plan dimension does not match spec.p_pad")
    if compute not in COMPUTE:
        raise ParameterError(f"compute must be 'f64' or 'f32', got {compute!r}")
    spec.gpu_kind()
    device = torch.device(device) if device is not None else default_device()
    if values_dtype is None:
        values_dtype = torch.float64 if compute == "f64" else torch.float32
    n = source.n
    given = indices is not None
    if given:
        idx_t = indices if isinstance(indices, torch.Tensor) else torch.from_numpy(np.asarray(indices).astype(np.int64))
        if tuple(idx_t.shape) != (n, plan.m):
            raise DimensionError(f"indices must be ({n}, {plan.m}), got {tuple(idx_t.shape)}")
        if n and (int(idx_t.min()) < 0 or int(idx_t.max()) >= spec.p_pad):
            raise DimensionError(f"indices must lie in [0, {spec.p_pad})")
        if n and plan.m > 1 and not bool((idx_t[:, 1:] > idx_t[:, :-1]).all()):
            raise DimensionError("each row of indices must be strictly increasing")
        indices = idx_t.to(device=device, dtype=torch.int32).contiguous()
    else:
        indices = torch.empty((n, plan.m), dtype=torch.int32, device=device)
    values = torch.empty((n, plan.m), dtype=values_dtype, device=device)
    row_iter = source.row_chunks() if hasattr(source, "row_chunks") else (ch.T for ch in source.chunks())
    j0 = 0
    for chunk in device_row_chunks(row_iter, device):
        rows = chunk
        if rows.ndim != 2 or rows.shape[1] != spec.p:
            raise DimensionError(
                f"bad chunk at column offset {j0}: expected ({spec.p}, c) block, got {tuple(rows.T.shape)}"
            )
        c = rows.shape[0]
        if j0 + c > n:
            raise DimensionError(f"source yielded more than {n} columns")
        if given:
            sketch_given_rows(rows, spec, plan.m, COMPUTE[compute], indices[j0 : j0 + c], values[j0 : j0 + c])
        else:
            _launch_rows(rows, spec, plan, col0 + j0, COMPUTE[compute], indices[j0 : j0 + c], values[j0 : j0 + c])
        j0 += c
    if j0 != n:
        raise DimensionError(f"source yielded {j0} columns, expected {n}")
    return SparseSketch(spec=spec, n=n, indices=indices, values=values, plan=plan, col0=int(col0))


def sketch_column(x, spec: PreconditionSpec, plan: SamplingPlan, i: int):
    """Sketch one column: (indices, values) of precondition(x) at indices(i); sketch.py:187-193"""
    if plan.p != spec.p_pad:
        raise DimensionError("plan dimension does not match spec.p_pad")
    t, host = as_device(x)
    if tuple(t.shape) != (spec.p,):
        raise DimensionError(f"expected length {spec.p}, got shape {tuple(t.shape)}")
    idx = torch.empty((1, plan.m), dtype=torch.int32, device=t.device)
    val = torch.empty((1, plan.m), dtype=torch.float64, device=t.device)
    _launch_rows(t[None, :], spec, plan, int(i), _lib.F64, idx, val)
    if host:
        return idx[0].cpu().numpy().astype(np.uint32), val[0].cpu().numpy()
    return idx[0], val[0]
