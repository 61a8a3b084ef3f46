"""DNSE1 dense matrices, SKCH1 sketches, and an out-of-core dense source.

Mirrors io.py:1-136 of the reference: the same byte formats and errors.
* DNSE1: magic ``b"DNSE1"``, little-endian u64 (p, n), then column-major f64. A column
  (one sample) is p contiguous f64, so a chunk of c columns is a row-major (c, p) block,
  the kernels' native layout.
* SKCH1: magic ``b"SKCH1"``, little-endian u64 (p_raw, p_pad, n, m, kind, sign_seed,
  master_seed), then per sample m u32 indices followed by m f64 values.

The GPU side stays in the device layout: ``DenseFileSource.row_chunks`` reads each chunk
straight into pinned host memory, and ``sketch_stream`` copies it ahead of the kernels
(``sketch.device_row_chunks``). ``write_sketch`` and ``read_sketch`` build and split the
SKCH1 record stream on the GPU (``skc_sketch_pack_records`` / ``..._unpack_records``), so
each chunk crosses PCIe in one copy.
"""

from __future__ import annotations

import struct
from typing import Iterator

import numpy as np
import torch

from . import _lib
from .errors import DimensionError, ParameterError
from .sketch import SamplingPlan, SparseSketch
from .transform import DCT, HADAMARD, NONE, PreconditionSpec, default_device

DENSE_MAGIC = b"DNSE1"
SKETCH_MAGIC = b"SKCH1"
FILE_KIND_CODES = {NONE: 0, HADAMARD: 1, DCT: 2}  # SKCH1 header codes (io.py:22-23)
FILE_KIND_NAMES = {v: k for k, v in FILE_KIND_CODES.items()}
_DENSE_HEADER = struct.Struct("<QQ")
_SKETCH_HEADER = struct.Struct("<7Q")
RECORD_CHUNK = 1 << 16  # samples per pack / unpack round trip


def _dense_header(fh, path) -> tuple[int, int]:
    magic = fh.read(len(DENSE_MAGIC))
    if magic != DENSE_MAGIC:
        raise DimensionError(f"not a DNSE1 file (magic {magic!r})")
    raw = fh.read(_DENSE_HEADER.size)
    if len(raw) != _DENSE_HEADER.size:
        raise DimensionError(f"truncated dense header: {path}")
    p, n = _DENSE_HEADER.unpack(raw)
    return int(p), int(n)


def write_dense(path, X) -> None:
    """Write a (p, n) matrix as DNSE1 (column-major f64); io.py:25-33"""
    X = np.asarray(X.cpu().numpy() if isinstance(X, torch.Tensor) else X, dtype=np.float64)
    if X.ndim != 2:
        raise DimensionError("expected a (p, n) matrix")
    with open(path, "wb") as fh:
        fh.write(DENSE_MAGIC)
        fh.write(_DENSE_HEADER.pack(X.shape[0], X.shape[1]))
        fh.write(np.asfortranarray(X).tobytes(order="F"))


def read_dense(path) -> np.ndarray:
    """Load a whole DNSE1 file as a (p, n) array; io.py:36-43"""
    with open(path, "rb") as fh:
        p, n = _dense_header(fh, path)
        data = np.fromfile(fh, dtype="<f8", count=p * n)
    if data.size != p * n:
        raise DimensionError(f"truncated dense file: {path}")
    return data.reshape((p, n), order="F")


class DenseFileSource:
    """Out-of-core column source over a DNSE1 file; io.py:54-81.

    ``chunks()`` yields (p, c) f64 column blocks like the reference. ``row_chunks()`` (used
    by ``sketch_stream``) yields the same bytes as pinned (c, p) torch tensors read
    straight from the file. Every pass reopens the file and counts in ``passes``.
    """

    def __init__(self, path, chunk_cols: int = 8192):
        if chunk_cols < 1:
            raise ParameterError("chunk_cols must be >= 1")
        self.path = path
        self.chunk_cols = int(chunk_cols)
        with open(path, "rb") as fh:
            self.p, self.n = _dense_header(fh, path)
        self.passes = 0

    def _blocks(self, pinned: bool) -> Iterator[np.ndarray]:
        self.passes += 1
        with open(self.path, "rb") as fh:
            _dense_header(fh, self.path)
            for j0 in range(0, self.n, self.chunk_cols):
                c = min(self.chunk_cols, self.n - j0)
                if pinned:
                    t = torch.empty((c, self.p), dtype=torch.float64, pin_memory=True)
                    buf = t.numpy()
                else:
                    t = None
                    buf = np.empty((c, self.p), dtype="<f8")
                got = fh.readinto(memoryview(buf).cast("B"))
                if got != buf.nbytes:
                    raise DimensionError(f"read failure at column offset {j0} of {self.path}")
                yield t if pinned else buf

    def chunks(self) -> Iterator[np.ndarray]:
        for rows in self._blocks(pinned=False):
            yield rows.T

    def row_chunks(self) -> Iterator[torch.Tensor]:
        return self._blocks(pinned=torch.cuda.is_available())


def _kind_code(spec: PreconditionSpec) -> int:
    return FILE_KIND_CODES[spec.kind]


def write_sketch(path, sketch: SparseSketch) -> None:
    """Write a SparseSketch as SKCH1 (bit-exact round trip); io.py:88-110.

    Records are packed on the GPU in chunks of RECORD_CHUNK samples and written from
    pinned memory.
    """
    spec, plan = sketch.spec, sketch.plan
    master = plan.master_seed if plan is not None else 0
    n, m = sketch.n, sketch.m
    dev = sketch.indices.device
    with open(path, "wb") as fh:
        fh.write(SKETCH_MAGIC)
        fh.write(_SKETCH_HEADER.pack(spec.p, spec.p_pad, n, m, _kind_code(spec), spec.sign_seed & 0xFFFFFFFFFFFFFFFF,
                                     master & 0xFFFFFFFFFFFFFFFF))
        if n == 0:
            return
        rows = min(n, RECORD_CHUNK)
        words = torch.empty((rows, 3 * m), dtype=torch.int32, device=dev)
        host = torch.empty((rows, 3 * m), dtype=torch.int32, pin_memory=True)
        vals = sketch.values.contiguous()
        idx = sketch.indices.contiguous()
        with torch.cuda.device(dev):
            for r0 in range(0, n, rows):
                c = min(rows, n - r0)
                _lib.call("skc_sketch_pack_records", idx[r0:].data_ptr(), vals[r0:].data_ptr(), _lib.dtype_code(vals),
                          c, m, words.data_ptr(), _lib.stream_ptr(dev))
                host[:c].copy_(words[:c])
                fh.write(memoryview(host[:c].numpy()).cast("B"))


def read_sketch(path, device=None) -> SparseSketch:
    """Read a SKCH1 file into a device SparseSketch (int32 indices, f64 values); io.py:113-136"""
    device = torch.device(device) if device is not None else default_device()
    with open(path, "rb") as fh:
        magic = fh.read(len(SKETCH_MAGIC))
        if magic != SKETCH_MAGIC:
            raise DimensionError(f"not a SKCH1 file (magic {magic!r})")
        raw = fh.read(_SKETCH_HEADER.size)
        if len(raw) != _SKETCH_HEADER.size:
            raise DimensionError(f"truncated sketch header: {path}")
        p_raw, p_pad, n, m, kind_code, sign_seed, master_seed = _SKETCH_HEADER.unpack(raw)
        if kind_code not in FILE_KIND_NAMES:
            raise DimensionError(f"unknown transform code {kind_code}")
        spec = PreconditionSpec(kind=FILE_KIND_NAMES[kind_code], sign_seed=int(sign_seed), p=int(p_raw),
                                p_pad=int(p_pad))
        plan = SamplingPlan(master_seed=int(master_seed), p=int(p_pad), m=int(m))
        n, m = int(n), int(m)
        idx = torch.empty((n, m), dtype=torch.int32, device=device)
        val = torch.empty((n, m), dtype=torch.float64, device=device)
        if n:
            rows = min(n, RECORD_CHUNK)
            host = torch.empty((rows, 3 * m), dtype=torch.int32, pin_memory=True)
            words = torch.empty((rows, 3 * m), dtype=torch.int32, device=device)
            with torch.cuda.device(device):
                for r0 in range(0, n, rows):
                    c = min(rows, n - r0)
                    buf = host[:c].numpy()
                    if fh.readinto(memoryview(buf).cast("B")) != buf.nbytes:
                        raise DimensionError(f"truncated sketch file: {path}")
                    words[:c].copy_(host[:c])
                    _lib.call("skc_sketch_unpack_records", words.data_ptr(), c, m, idx[r0:].data_ptr(),
                              val[r0:].data_ptr(), _lib.stream_ptr(device))
                    torch.cuda.current_stream(device).synchronize()  # host buffer is refilled next
    return SparseSketch(spec=spec, n=n, indices=idx, values=val, plan=plan)


__all__ = ["DENSE_MAGIC", "SKETCH_MAGIC", "DenseFileSource", "read_dense", "read_sketch", "write_dense",
           "write_sketch"]
