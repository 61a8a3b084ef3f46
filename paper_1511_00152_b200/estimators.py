"""Unbiased mean / covariance estimators and PCA on a GPU sketch; estimators.py:1-129.

Device work per estimate:
  K2 ``skc_moments``         mean accumulation + value statistics
  K3 ``skc_cov_accumulate``  raw W W^T upper triangle (fixed-point smem bands)
  K4 ``skc_cov_finalize``    scale, symmetrise, diagonal debias
  K7 ``skc_mean_finalize`` / ``skc_unprecondition``  adjoint transforms
The top-k eigensolve is handed back to the host (numpy LAPACK ``eigh``), as the
north star specifies. Partial sums (acc, stats, triangle) are plain device tensors, so
a sharded run allreduces them between accumulate and finalize (``dist.py``).
"""

from __future__ import annotations

from dataclasses import dataclass, field
from typing import Optional

import numpy as np
import torch

from . import _lib
from .errors import DimensionError, ParameterError
from .sketch import SparseSketch
from .transform import default_device, u64, unprecondition

SYMMETRY_RTOL = 1e-9


@dataclass
class CovarianceEstimate:
    """Symmetric p_pad x p_pad estimate; estimators.py:21-27. ``matrix`` is host numpy,
    ``device_matrix`` the same values on the GPU."""

    matrix: np.ndarray
    n_used: int
    domain: str = "preconditioned"
    device_matrix: Optional[torch.Tensor] = field(default=None, repr=False)


@dataclass
class Moments:
    """Device partial sums of one sketch (or one shard): mean accumulator, stats, triangle.

    ``packed`` is one contiguous fp64 buffer [acc (p_pad) | stats (3) | tri] of which acc,
    stats and tri are views, so a sharded run combines all partials with ONE allreduce
    (dist.combine_moments; "parallel partial sums then ordered combine")."""

    acc: torch.Tensor    # (p_pad,) fp64
    stats: torch.Tensor  # (3,) fp64: sum v^2, max |v|, rows
    tri: Optional[torch.Tensor]  # (p_pad (p_pad+1)/2,) fp64 or None
    n: int
    packed: Optional[torch.Tensor] = None

    @classmethod
    def zeros(cls, p_pad: int, covariance: bool, device) -> "Moments":
        tri_len = p_pad * (p_pad + 1) // 2 if covariance else 0
        buf = torch.zeros(p_pad + 3 + tri_len, dtype=torch.float64, device=device)
        return cls(acc=buf[:p_pad], stats=buf[p_pad:p_pad + 3], tri=buf[p_pad + 3:] if covariance else None, n=0,
                   packed=buf)


def accumulate_moments(sketch: SparseSketch, covariance: bool = True, into: Optional[Moments] = None) -> Moments:
    """K2 (+ K3) over one sketch; adds into ``into`` when given (chunked / sharded use)."""
    dev = sketch.indices.device
    p, m, n = sketch.p, sketch.m, sketch.n
    if into is None:
        into = Moments.zeros(p, covariance, dev)
    L = _lib.lib()
    st = _lib.stream_ptr(dev)
    vcode = _lib.dtype_code(sketch.values)
    idx, val = sketch.indices.contiguous(), sketch.values.contiguous()
    with torch.cuda.device(dev):
        ws = _lib.workspace(L.skc_moments_workspace(n, m, p), dev)
        _lib.call("skc_moments", idx.data_ptr(), val.data_ptr(), vcode, n, m, p, into.acc.data_ptr(),
                  into.stats.data_ptr(), ws.data_ptr(), ws.numel(), st)
        if covariance:
            ws2 = _lib.workspace(L.skc_cov_workspace(n, m, p), dev)
            _lib.call("skc_cov_accumulate", idx.data_ptr(), val.data_ptr(), vcode, n, m, p, into.stats.data_ptr(),
                      into.tri.data_ptr(), ws2.data_ptr(), ws2.numel(), st)
    into.n += n
    return into


def stream_moments(source, spec, plan, *, covariance: bool = True, compute: str = "f64", device=None,
                   col0: int = 0, into: Optional[Moments] = None) -> Moments:
    """Sketch and accumulate the estimators' partial sums chunk by chunk, without keeping the
    sketch (sketch.py:196-223 then estimators.py:30-66).

    Host chunks reach the device through pinned, double-buffered copies on a copy stream
    (``sketch.device_row_chunks``). Each chunk's K1 / K2 / K3 run on the compute stream while
    the next chunk is in flight, so an end-to-end covariance from host data runs at the
    PCIe rate. K3's fixed-point scale follows the statistics accumulated so far; every
    chunk's sum is exact in its own quantum and the chunks add in fp64.
    """
    from .sketch import COMPUTE, RowSource, _launch_rows, as_source, device_row_chunks

    source = as_source(source)
    if source.p != spec.p:
        raise DimensionError(f"source has p={source.p}, spec expects {spec.p}")
    if compute not in COMPUTE:
        raise ParameterError(f"compute must be 'f64' or 'f32', got {compute!r}")
    device = torch.device(device) if device is not None else default_device()
    vdt = torch.float64 if compute == "f64" else torch.float32
    rows = getattr(source, "rows", None)
    if (isinstance(source, RowSource) and isinstance(rows, torch.Tensor) and not rows.is_cuda and rows.is_pinned()
            and rows.dtype in (torch.float32, torch.float64) and rows.ndim == 2 and rows.stride(1) == 1):
        return _stream_moments_native(rows, source.chunk_cols, spec, plan, covariance, compute, device, col0, into)
    row_iter = source.row_chunks() if hasattr(source, "row_chunks") else (ch.T for ch in source.chunks())
    j0 = 0
    for rows in device_row_chunks(row_iter, device):
        if rows.ndim != 2 or rows.shape[1] != spec.p:
            raise DimensionError(f"bad chunk at column offset {j0}: expected ({spec.p}, c)")
        c = rows.shape[0]
        idx = torch.empty((c, plan.m), dtype=torch.int32, device=device)
        val = torch.empty((c, plan.m), dtype=vdt, device=device)
        _launch_rows(rows, spec, plan, col0 + j0, COMPUTE[compute], idx, val)
        sk = SparseSketch(spec=spec, n=c, indices=idx, values=val, plan=plan, col0=col0 + j0)
        into = accumulate_moments(sk, covariance=covariance, into=into)
        j0 += c
    if j0 != source.n:
        raise DimensionError(f"source yielded {j0} columns, expected {source.n}")
    if into is None:
        raise ParameterError("empty source")
    return into


def _stream_moments_native(rows: torch.Tensor, chunk_rows: int, spec, plan, covariance: bool, compute: str, device,
                           col0: int, into: Optional[Moments]) -> Moments:
    """Pinned host rows: the chunk loop runs in C++ (``skc_stream_moments``): copies on a
    private stream into two device buffers, each chunk's kernels on the current stream."""
    from .sketch import COMPUTE

    n, p = rows.shape
    p_pad, m = spec.p_pad, plan.m
    if into is None:
        into = Moments.zeros(p_pad, covariance, device)
    chunk = max(1, min(int(chunk_rows), max(int(n), 1)))
    L = _lib.lib()
    xc = _lib.dtype_code(rows)
    ws = _lib.workspace(L.skc_stream_workspace(chunk, p, p_pad, m, xc, COMPUTE[compute], int(covariance)), device)
    with torch.cuda.device(device):
        _lib.call("skc_stream_moments", rows.data_ptr(), xc, rows.stride(0), n, p, p_pad, spec.gpu_kind(),
                  u64(spec.sign_seed), u64(plan.master_seed), int(col0), m, COMPUTE[compute],
                  1 if plan.sampler == "philox" else 0, chunk, into.acc.data_ptr(), into.stats.data_ptr(),
                  _lib.ptr(into.tri), ws.data_ptr(), ws.numel(), _lib.stream_ptr(device))
    into.n += int(n)
    return into


def mean_from_moments(mom: Moments, spec, m: int, n_total: int) -> torch.Tensor:
    out = torch.empty(spec.p, dtype=torch.float64, device=mom.acc.device)
    with torch.cuda.device(out.device):
        _lib.call("skc_mean_finalize", mom.acc.data_ptr(), spec.p, spec.p_pad, m, int(n_total), spec.gpu_kind(),
                  u64(spec.sign_seed), out.data_ptr(), _lib.stream_ptr(out.device))
    return out


def covariance_from_moments(mom: Moments, p_pad: int, m: int, n_total: int) -> torch.Tensor:
    C = torch.empty((p_pad, p_pad), dtype=torch.float64, device=mom.tri.device)
    with torch.cuda.device(C.device):
        _lib.call("skc_cov_finalize", mom.tri.data_ptr(), p_pad, m, int(n_total), C.data_ptr(),
                  _lib.stream_ptr(C.device))
    return C


def estimate_mean(sketch: SparseSketch) -> np.ndarray:
    """(p/m)(1/n) sum of sketch columns, adjoint, truncate; estimators.py:30-45"""
    if sketch.n < 1:
        raise ParameterError("empty sketch")
    mom = accumulate_moments(sketch, covariance=False)
    return mean_from_moments(mom, sketch.spec, sketch.m, sketch.n).cpu().numpy()


def estimate_covariance(sketch: SparseSketch) -> CovarianceEstimate:
    """Unbiased covariance of the preconditioned data; estimators.py:48-66"""
    if sketch.m < 2:
        raise ParameterError("covariance estimation needs m >= 2")
    if sketch.n < 1:
        raise ParameterError("empty sketch")
    mom = accumulate_moments(sketch, covariance=True)
    C = covariance_from_moments(mom, sketch.p, sketch.m, sketch.n)
    return CovarianceEstimate(matrix=C.cpu().numpy(), n_used=sketch.n, device_matrix=C)


def top_eigenvectors(C, k: int, solver: str = "host"):
    """Eigenvectors of the k largest eigenvalues as columns; estimators.py:69-81.

    ``solver="host"`` (default) runs LAPACK ``eigh`` through numpy, exactly as the reference.
    ``solver="device"`` keeps C on the GPU and computes only the k largest eigenpairs
    (``skc_top_eigenvectors``: cuSOLVER syevdx over an index range), returning a CUDA tensor:
    the same eigenvectors up to each one's sign, within the eigensolver's rounding (SURVEY 8(f)
    row 2). Both check symmetry as the reference does.
    """
    if solver not in ("host", "device"):
        raise ParameterError(f"unknown solver {solver!r}")
    if solver == "device":
        Cd = C if isinstance(C, torch.Tensor) else torch.as_tensor(np.asarray(C, dtype=np.float64))
        Cd = Cd.to(dtype=torch.float64, device=Cd.device if Cd.is_cuda else default_device()).contiguous()
        if Cd.ndim != 2 or Cd.shape[0] != Cd.shape[1]:
            raise ParameterError("expected a square matrix")
        p = Cd.shape[0]
        if not 1 <= k <= p:
            raise ParameterError(f"need 1 <= k <= {p}, got {k}")
        scale = max(float(Cd.abs().max()), 1e-300)
        if float((Cd - Cd.T).abs().max()) > SYMMETRY_RTOL * scale:
            raise ParameterError("matrix is not symmetric within tolerance")
        L = _lib.lib()
        V = torch.empty((p, k), dtype=torch.float64, device=Cd.device)
        with torch.cuda.device(Cd.device):
            ws = _lib.workspace(L.skc_top_eigenvectors_workspace(p, k), Cd.device)
            _lib.call("skc_top_eigenvectors", Cd.data_ptr(), p, k, V.data_ptr(), None, ws.data_ptr(), ws.numel(),
                      _lib.stream_ptr(Cd.device))
        return V
    C = C.cpu().numpy() if isinstance(C, torch.Tensor) else np.asarray(C, dtype=np.float64)
    if C.ndim != 2 or C.shape[0] != C.shape[1]:
        raise ParameterError("expected a square matrix")
    p = C.shape[0]
    if not 1 <= k <= p:
        raise ParameterError(f"need 1 <= k <= {p}, got {k}")
    scale = max(float(np.abs(C).max()), 1e-300)
    if np.abs(C - C.T).max() > SYMMETRY_RTOL * scale:
        raise ParameterError("matrix is not symmetric within tolerance")
    w, V = np.linalg.eigh(0.5 * (C + C.T))
    return V[:, ::-1][:, :k]


def principal_components(sketch: SparseSketch, k: int, solver: str = "host") -> np.ndarray:
    """Top-k PCs mapped back to the original domain; estimators.py:116-129.

    The adjoint (FWHT then D, truncation) runs on the device for all k vectors at once;
    ``solver`` selects the host (reference) or device eigensolve.
    """
    est = estimate_covariance(sketch)
    spec = sketch.spec
    if solver == "device":
        Vd = top_eigenvectors(est.device_matrix, k, solver="device").T.contiguous()
    else:
        V = top_eigenvectors(est.matrix, k)
        Vd = torch.as_tensor(np.ascontiguousarray(V.T), device=sketch.indices.device)
    U = torch.empty((k, spec.p), dtype=torch.float64, device=Vd.device)
    with torch.cuda.device(Vd.device):
        _lib.call("skc_unprecondition", Vd.data_ptr(), k, spec.p_pad, spec.gpu_kind(), u64(spec.sign_seed), spec.p,
                  U.data_ptr(), _lib.stream_ptr(Vd.device))
    return U.T.contiguous().cpu().numpy()


__all__ = [
    "CovarianceEstimate", "Moments", "SYMMETRY_RTOL", "accumulate_moments", "covariance_from_moments",
    "stream_moments",
    "estimate_covariance", "estimate_mean", "mean_from_moments", "principal_components", "top_eigenvectors",
    "unprecondition",
]
