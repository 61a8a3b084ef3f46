"""Orthonormal preconditioner x -> H D x and its adjoint, on the GPU.

Mirrors transform.py:1-200 of the reference (``PreconditionSpec``, ``precondition``,
``unprecondition``, the ``_columns`` variants, ``fwht_inplace``, ``next_pow2``). The
arithmetic runs in fp64 in the reference's butterfly order, through ``skc_precondition``
/ ``skc_unprecondition`` / ``skc_fwht``, so results are bit-identical. I/O follows one
rule throughout: numpy in gives numpy out, and a CUDA tensor in gives a CUDA tensor
out on the same device. The DCT kind is outside the GPU hot path: creating a DCT spec
is allowed, as in the reference, but transforming with it raises ParameterError.
"""

from __future__ import annotations

from dataclasses import dataclass
from functools import lru_cache

import numpy as np
import torch

from . import _lib
from .errors import DimensionError, ParameterError

HADAMARD = "hadamard"
DCT = "dct"
NONE = "none"
KINDS = (HADAMARD, DCT, NONE)


def next_pow2(n: int) -> int:
    """transform.py:26-27"""
    return 1 << (int(n) - 1).bit_length()


def u64(x: int) -> int:
    return int(x) & 0xFFFFFFFFFFFFFFFF


def default_device() -> torch.device:
    """The current CUDA device; raises DeviceError when there is none (no CPU fallback)."""
    if not torch.cuda.is_available():
        from .errors import DeviceError

        raise DeviceError("no CUDA device: the sketch hot path runs only on the GPU")
    return torch.device("cuda", torch.cuda.current_device())


@dataclass(frozen=True)
class PreconditionSpec:
    """Transform kind, sign seed and (original, padded) dimensions; transform.py:30-75."""

    kind: str
    sign_seed: int
    p: int
    p_pad: int

    def __post_init__(self):
        if self.kind not in KINDS:
            raise ParameterError(f"unknown transform kind {self.kind!r}")
        if self.p < 1:
            raise DimensionError("dimension must be positive")
        if self.p_pad < self.p:
            raise DimensionError("padded dimension smaller than original")
        if self.kind == HADAMARD and self.p_pad & (self.p_pad - 1):
            raise DimensionError("hadamard padded dimension must be a power of two")
        if self.kind != HADAMARD and self.p_pad != self.p:
            raise DimensionError(f"{self.kind} transform does not pad")

    @classmethod
    def create(cls, kind: str, p: int, sign_seed: int = 0) -> "PreconditionSpec":
        p_pad = next_pow2(p) if kind == HADAMARD else p
        return cls(kind=kind, sign_seed=int(sign_seed), p=int(p), p_pad=p_pad)

    @property
    def eta(self) -> float:
        if self.kind == HADAMARD:
            return 1.0
        if self.kind == DCT:
            return 0.5
        raise ParameterError("eta is undefined for the identity preconditioner")

    @property
    def kind_code(self) -> int:
        return _lib.KIND_CODES[self.kind]

    def gpu_kind(self) -> int:
        if self.kind == DCT:
            raise ParameterError("the dct preconditioner is not on the GPU hot path (hadamard or none)")
        return self.kind_code

    def device_signs(self, device=None) -> torch.Tensor:
        """D diagonal as a CUDA fp64 tensor, generated on the device (_hash.py:38-43)."""
        device = torch.device(device) if device is not None else default_device()
        out = torch.empty(self.p_pad, dtype=torch.float64, device=device)
        with torch.cuda.device(device):
            _lib.call("skc_signs", u64(self.sign_seed), self.p_pad, self.gpu_kind(), out.data_ptr(),
                      _lib.stream_ptr(device))
        return out

    def signs(self) -> np.ndarray:
        """The +-1 diagonal of D, length p_pad (read-only, cached); transform.py:71-75"""
        return _cached_signs(self.kind, u64(self.sign_seed), self.p_pad)


@lru_cache(maxsize=128)
def _cached_signs(kind: str, sign_seed: int, p_pad: int) -> np.ndarray:
    s = PreconditionSpec(kind, sign_seed, p_pad, p_pad).device_signs().cpu().numpy()
    s.setflags(write=False)
    return s


# ---- host/device I/O ---------------------------------------------------------------

def as_device(x, dtype=None, device=None) -> tuple[torch.Tensor, bool]:
    """Return (CUDA tensor, came_from_host). Keeps float32 / float64; casts other dtypes to fp64."""
    if isinstance(x, torch.Tensor):
        t = x
        host = not t.is_cuda
    else:
        t = torch.from_numpy(np.ascontiguousarray(np.asarray(x)))
        host = True
    if dtype is not None:
        t = t.to(dtype)
    elif t.dtype not in (torch.float32, torch.float64):
        t = t.to(torch.float64)
    if not t.is_cuda:
        t = t.to(device if device is not None else default_device(), non_blocking=False)
    return t, host


def _out(t: torch.Tensor, host: bool):
    return t.cpu().numpy() if host else t


def _rows_transform(rows: torch.Tensor, spec: PreconditionSpec) -> torch.Tensor:
    """(c, p) rows on the device -> (c, p_pad) fp64 rows of H D pad(x)."""
    rows = rows.contiguous()
    c = rows.shape[0]
    Y = torch.empty((c, spec.p_pad), dtype=torch.float64, device=rows.device)
    with torch.cuda.device(rows.device):
        _lib.call("skc_precondition", rows.data_ptr(), _lib.dtype_code(rows), spec.p, c, spec.p, spec.p_pad,
                  spec.gpu_kind(), u64(spec.sign_seed), Y.data_ptr(), _lib.stream_ptr(rows.device))
    return Y


def _rows_adjoint(rows: torch.Tensor, spec: PreconditionSpec, p_out: int) -> torch.Tensor:
    rows = rows.to(torch.float64).contiguous()
    c = rows.shape[0]
    X = torch.empty((c, p_out), dtype=torch.float64, device=rows.device)
    with torch.cuda.device(rows.device):
        _lib.call("skc_unprecondition", rows.data_ptr(), c, spec.p_pad, spec.gpu_kind(), u64(spec.sign_seed), p_out,
                  X.data_ptr(), _lib.stream_ptr(rows.device))
    return X


def precondition(x, spec: PreconditionSpec):
    """Length-p vector -> H D pad(x), length p_pad; transform.py:157-166"""
    t, host = as_device(x)
    if tuple(t.shape) != (spec.p,):
        raise DimensionError(f"expected length {spec.p}, got shape {tuple(t.shape)}")
    return _out(_rows_transform(t[None, :], spec)[0], host)


def unprecondition(y, spec: PreconditionSpec):
    """Adjoint D^T H^T, the exact inverse of ``precondition``; transform.py:169-177"""
    t, host = as_device(y, torch.float64)
    if tuple(t.shape) != (spec.p_pad,):
        raise DimensionError(f"expected length {spec.p_pad}, got shape {tuple(t.shape)}")
    return _out(_rows_adjoint(t[None, :], spec, spec.p_pad)[0], host)


def precondition_columns(X, spec: PreconditionSpec):
    """Precondition every column of a (p, c) block; returns (p_pad, c). transform.py:180-189"""
    t, host = as_device(X)
    if t.ndim != 2 or t.shape[0] != spec.p:
        raise DimensionError(f"expected ({spec.p}, c) block, got {tuple(t.shape)}")
    return _out(_rows_transform(t.T, spec).T.contiguous(), host)


def unprecondition_columns(Y, spec: PreconditionSpec):
    """Adjoint of ``precondition_columns`` on a (p_pad, c) block; transform.py:192-200"""
    t, host = as_device(Y, torch.float64)
    if t.ndim != 2 or t.shape[0] != spec.p_pad:
        raise DimensionError(f"expected ({spec.p_pad}, c) block, got {tuple(t.shape)}")
    return _out(_rows_adjoint(t.T, spec, spec.p_pad).T.contiguous(), host)


def fwht_inplace(v):
    """Orthonormal WHT of a power-of-two-length vector, overwriting v; transform.py:113-122"""
    t, host = as_device(v, torch.float64)
    if t.ndim != 1:
        raise DimensionError("fwht_inplace expects a vector")
    p = t.shape[0]
    if p < 1 or p & (p - 1):
        raise DimensionError(f"length {p} is not a power of two")
    out = torch.empty_like(t)
    with torch.cuda.device(t.device):
        _lib.call("skc_fwht", t.data_ptr(), 1, p, out.data_ptr(), _lib.stream_ptr(t.device))
    if host:
        res = out.cpu().numpy()
        if isinstance(v, np.ndarray) and v.dtype == np.float64:
            v[...] = res
            return v
        return res
    if isinstance(v, torch.Tensor) and v.is_cuda and v.dtype == torch.float64:
        v.copy_(out)
        return v
    return out
