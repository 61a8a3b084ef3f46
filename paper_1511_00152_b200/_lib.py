"""ctypes binding of libsketchcu.so, the C ABI declared in include/sketchcu.h.

The product path runs only through this library. If the library is missing, or no
CUDA device is present, every call raises DeviceError. There is no CPU fallback.
"""

from __future__ import annotations

import ctypes
import os
import threading

import torch

from .errors import CommError, DeviceError, DimensionError, ParameterError

_HERE = os.path.dirname(os.path.abspath(__file__))
# SKC_LIB selects an alternative build of the same library (kernel A/B experiments)
SO_PATH = os.environ.get("SKC_LIB") or os.path.join(_HERE, "_lib", "libsketchcu.so")

SKC_OK, SKC_EDIM, SKC_EPARAM, SKC_ECUDA, SKC_ENCCL = 0, 1, 2, 3, 4
KIND_CODES = {"hadamard": 0, "dct": 1, "none": 2}
F32, F64 = 0, 1

_c = ctypes
_P, _I32, _I64, _U64, _SZ = _c.c_void_p, _c.c_int32, _c.c_int64, _c.c_uint64, _c.c_size_t

# name -> (restype, argtypes)
SIGNATURES = {
    "skc_last_error": (_c.c_char_p, []),
    "skc_abi_version": (_c.c_int, []),
    "skc_max_p_pad": (_I32, []),
    "skc_launch_count": (_U64, []),
    "skc_count_launches": (None, [_U64]),
    "skc_kmeans_lloyd_workspace": (_SZ, [_I64, _I32, _I32, _I32, _I32, _I32]),
    "skc_kmeans_lloyd": (_c.c_int, [_P, _P, _I32, _I64, _I32, _I32, _I32, _P, _I32, _P, _P, _P, _SZ, _P, _P, _P, _P,
                                    _P]),
    "skc_kmeans_lloyd_graph_kernels": (None, [_P, _P]),
    "skc_kmeans_assign_one": (_c.c_int, [_P, _P, _I32, _I32, _P, _I32, _I32, _P, _P, _P]),
    "skc_row_sqnorms": (_c.c_int, [_P, _I32, _I64, _I32, _P, _P]),
    "skc_kmeans_d2_to_point": (_c.c_int, [_P, _P, _I32, _I64, _I32, _I32, _I64, _P, _P, _P, _P]),
    "skc_kmeans_d2_to_dense": (_c.c_int, [_P, _P, _I32, _I64, _I32, _I32, _P, _P, _P, _P, _P]),
    "skc_signs": (_c.c_int, [_U64, _I32, _I32, _P, _P]),
    "skc_precondition": (_c.c_int, [_P, _I32, _I64, _I64, _I32, _I32, _I32, _U64, _P, _P]),
    "skc_unprecondition": (_c.c_int, [_P, _I64, _I32, _I32, _U64, _I32, _P, _P]),
    "skc_fwht": (_c.c_int, [_P, _I64, _I32, _P, _P]),
    "skc_indices": (_c.c_int, [_U64, _I64, _I64, _I32, _I32, _P, _P]),
    "skc_sketch": (_c.c_int, [_P, _I32, _I64, _I64, _I32, _I32, _I32, _U64, _U64, _I64, _I32, _I32, _P, _P, _I32,
                              _P]),
    "skc_moments_workspace": (_SZ, [_I64, _I32, _I32]),
    "skc_moments": (_c.c_int, [_P, _P, _I32, _I64, _I32, _I32, _P, _P, _P, _SZ, _P]),
    "skc_mean_finalize": (_c.c_int, [_P, _I32, _I32, _I32, _I64, _I32, _U64, _P, _P]),
    "skc_cov_workspace": (_SZ, [_I64, _I32, _I32]),
    "skc_cov_accumulate": (_c.c_int, [_P, _P, _I32, _I64, _I32, _I32, _P, _P, _P, _SZ, _P]),
    "skc_cov_finalize": (_c.c_int, [_P, _I32, _I32, _I64, _P, _P]),
    "skc_kmeans_init": (_c.c_int, [_P, _P, _I32, _I64, _I32, _P, _I32, _I32, _P, _P]),
    "skc_kmeans_assign_workspace": (_SZ, [_I64, _I32, _I32]),
    "skc_kmeans_assign": (_c.c_int, [_P, _P, _I32, _I64, _I32, _P, _I32, _I32, _P, _P, _P, _P, _P, _P, _SZ, _P]),
    "skc_kmeans_tc_supported": (_c.c_int, [_I32, _I32, _I32]),
    "skc_kmeans_tc_prepare_workspace": (_SZ, [_I64, _I32, _I32]),
    "skc_kmeans_tc_prepare": (_c.c_int, [_P, _P, _I32, _I64, _I32, _I32, _P, _SZ, _P]),
    "skc_kmeans_assign_tc_workspace": (_SZ, [_I64, _I32, _I32]),
    "skc_kmeans_assign_tc": (_c.c_int, [_P, _P, _I32, _I64, _I32, _P, _I32, _I32, _P, _P, _P, _P, _P, _P, _P, _SZ,
                                        _P]),
    "skc_pairwise_sum_workspace": (_SZ, [_I64]),
    "skc_pairwise_sum": (_c.c_int, [_P, _I64, _P, _P, _SZ, _P]),
    "skc_kmeans_partials_workspace": (_SZ, [_I64, _I32, _I32, _I32]),
    "skc_kmeans_partials": (_c.c_int, [_P, _P, _I32, _I64, _I32, _P, _I32, _I32, _P, _P, _P, _P, _SZ, _P]),
    "skc_kmeans_centers": (_c.c_int, [_P, _P, _P, _P, _I32, _I32, _P, _P, _P]),
    "skc_kmeans_reseed": (_c.c_int, [_P, _P, _I32, _I32, _P, _I32, _I32, _P, _P]),
    "skc_kmeans_csc_workspace": (_c.c_size_t, [_I64, _I32, _I32, _I32]),
    "skc_kmeans_build_csc": (_c.c_int, [_P, _P, _I32, _I64, _I32, _I32, _P, _SZ, _P]),
    "skc_kmeans_seg_workspace": (_c.c_size_t, [_I64, _I32, _I32, _I32, _I32]),
    "skc_kmeans_partials_csc": (_c.c_int, [_P, _I32, _I64, _I32, _I32, _P, _I32, _P, _P, _P, _P, _SZ, _P]),
    "skc_kmeans_reseed_at": (_c.c_int, [_P, _P, _I32, _I64, _I32, _P, _P, _I32, _I32, _P, _P]),
    "skc_indices_philox": (_c.c_int, [_U64, _I64, _I64, _I32, _I32, _P, _P]),
    "skc_sketch_given": (_c.c_int, [_P, _I32, _I64, _I64, _I32, _I32, _I32, _U64, _I32, _I32, _P, _P, _I32, _P]),
    "skc_stream_workspace": (_c.c_size_t, [_I64, _I32, _I32, _I32, _I32, _I32, _I32]),
    "skc_stream_moments": (_c.c_int, [_P, _I32, _I64, _I64, _I32, _I32, _I32, _U64, _U64, _I64, _I32, _I32, _I32, _I64,
                                      _P, _P, _P, _P, _SZ, _P]),
    "skc_sketch_pack_records": (_c.c_int, [_P, _P, _I32, _I64, _I32, _P, _P]),
    "skc_sketch_unpack_records": (_c.c_int, [_P, _I64, _I32, _P, _P, _P]),
    "skc_top_eigenvectors_workspace": (_SZ, [_I32, _I32]),
    "skc_top_eigenvectors": (_c.c_int, [_P, _I32, _I32, _P, _P, _P, _SZ, _P]),
    "skc_nccl_get_unique_id": (_c.c_int, [_P]),
    "skc_nccl_comm_init_rank": (_c.c_int, [_P, _I32, _P, _I32]),
    "skc_nccl_comm_destroy": (_c.c_int, [_P]),
    "skc_allreduce_sum_f64": (_c.c_int, [_P, _SZ, _P, _P]),
    "skc_moments_packed_len": (_SZ, [_I32, _I32]),
    "skc_kmeans_exchange_len": (_SZ, [_I32, _I32, _I32]),
    "skc_kmeans_pack_exchange": (_c.c_int, [_P, _P, _P, _P, _P, _P, _I32, _I32, _I32, _I32, _I64, _P, _P]),
    "skc_kmeans_unpack_exchange": (_c.c_int, [_P, _I32, _I32, _P, _P, _P, _P]),
    "skc_dense_assign_workspace": (_c.c_size_t, [_I32, _I32]),
    "skc_dense_assign": (_c.c_int, [_P, _I32, _I64, _I64, _I32, _P, _I32, _P, _P, _P, _P]),
    "skc_dense_sums_workspace": (_c.c_size_t, [_I64, _I32, _I32]),
    "skc_dense_sums": (_c.c_int, [_P, _I32, _I64, _I64, _I32, _P, _I32, _P, _P, _P, _P]),
}

_lock = threading.Lock()
_lib = None


def load_library(path: str = SO_PATH):
    """dlopen the shared library and declare every exported signature (no GPU needed)."""
    global _lib
    with _lock:
        if _lib is None:
            if not os.path.exists(path):
                raise DeviceError(
                    f"{path} is missing: build it with `python -m paper_1511_00152_b200._build` "
                    "(the GPU path has no CPU fallback)"
                )
            L = ctypes.CDLL(path)
            for name, (res, args) in SIGNATURES.items():
                fn = getattr(L, name)
                fn.restype = res
                fn.argtypes = args
            _lib = L
    return _lib


def lib():
    L = load_library()
    if not torch.cuda.is_available():
        raise DeviceError("no CUDA device: the sketch hot path runs only on the GPU")
    return L


def check(rc: int) -> None:
    if rc == SKC_OK:
        return
    msg = (_lib.skc_last_error() or b"").decode(errors="replace") if _lib is not None else ""
    if rc == SKC_EDIM:
        raise DimensionError(msg)
    if rc == SKC_EPARAM:
        raise ParameterError(msg)
    if rc == SKC_ENCCL:
        raise CommError(msg)
    raise DeviceError(msg)


def call(name: str, *args):
    """Invoke an ABI entry point on the current torch stream and map its status code."""
    check(getattr(lib(), name)(*args))


def stream_ptr(device=None) -> int:
    return torch.cuda.current_stream(device).cuda_stream


def ptr(t) -> int:
    if t is None:
        return 0
    return t.data_ptr()


def dtype_code(t: torch.Tensor) -> int:
    if t.dtype == torch.float32:
        return F32
    if t.dtype == torch.float64:
        return F64
    raise ParameterError(f"unsupported dtype {t.dtype}")


def workspace(nbytes: int, device) -> torch.Tensor:
    return torch.empty(max(int(nbytes), 1), dtype=torch.uint8, device=device)
