"""CPU oracle. This is test infrastructure only, not a product path.

ctypes bindings over ``liboracle.so``, the plain-C restatement of the reference
hot path, plus the numpy glue that mirrors the reference's estimator and K-means
finalisation. Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s
CPU-baseline legs may import this module, and only as a checker or baseline.

Every function cites the reference ``file:line`` it restates. All paths are
relative to ``/root/reference/pkg/src/sketchpipe``. Parity is pinned by
``tests/test_oracle_golden.py`` against fixtures produced by running the
reference (``tests/golden/make_golden.py``).

Layout convention: sample-major rows. ``X[i]`` is column i of the reference's
``(p, n)`` matrix.
"""

from __future__ import annotations

import ctypes
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SO = os.path.join(_HERE, "liboracle.so")

HADAMARD, DCT, NONE = 0, 1, 2
KIND_CODES = {"hadamard": HADAMARD, "dct": DCT, "none": NONE}


def build() -> str:
    """Compile the C restatement in place (make). Returns the .so path."""
    subprocess.run(["make", "-s", "-C", _HERE], check=True)
    return _SO


_lib = None


def lib():
    global _lib
    if _lib is None:
        if not os.path.exists(_SO) or os.path.getmtime(_SO) < os.path.getmtime(
            os.path.join(_HERE, "sketch_oracle.c")
        ):
            build()
        L = ctypes.CDLL(_SO)
        u64, i64, i32 = ctypes.c_uint64, ctypes.c_int64, ctypes.c_int32
        P = ctypes.c_void_p
        L.orc_mix64.restype = u64
        L.orc_mix64.argtypes = [u64]
        L.orc_derive_seed.restype = u64
        L.orc_derive_seed.argtypes = [u64, u64]
        L.orc_signs.argtypes = [u64, i32, P]
        L.orc_column_keys.argtypes = [u64, i64, i64, i32, P]
        L.orc_indices_block.argtypes = [u64, i64, i64, i32, i32, P]
        L.orc_philox_indices.argtypes = [u64, i64, i64, i32, i32, P]
        L.orc_philox4x32_10.argtypes = [P, ctypes.c_uint32, ctypes.c_uint32]
        L.orc_fwht.argtypes = [P, i32]
        L.orc_precondition_rows.argtypes = [P, i64, i64, i32, i32, i32, u64, P]
        L.orc_unprecondition_rows.argtypes = [P, i64, i32, i32, u64, P]
        L.orc_sketch.argtypes = [P, i32, i64, i64, i32, i32, i32, u64, u64, i64, i32, P, P, i32]
        L.orc_mean_acc.argtypes = [P, P, i64, i32, i32, P]
        L.orc_cov_acc.argtypes = [P, P, i64, i32, i32, P, i32]
        L.orc_pairwise_sum.restype = ctypes.c_double
        L.orc_pairwise_sum.argtypes = [P, i64]
        L.orc_kmeans_assign.argtypes = [P, P, i64, i32, P, i32, i32, P, P, i32]
        L.orc_kmeans_update.argtypes = [P, P, i64, i32, P, i32, i32, P, P, P, P]
        _lib = L
    return _lib


def _p(a: np.ndarray):
    return a.ctypes.data_as(ctypes.c_void_p)


def _u64(x) -> int:
    return int(x) & 0xFFFFFFFFFFFFFFFF


# ---- L0 hash streams (_hash.py) -------------------------------------------------

def mix64(z: int) -> int:
    """_hash.py:20-26"""
    return int(lib().orc_mix64(_u64(z)))


def derive_seed(seed: int, tag: int) -> int:
    """_hash.py:33-35"""
    return int(lib().orc_derive_seed(_u64(seed), _u64(tag)))


def signs(sign_seed: int, p: int) -> np.ndarray:
    """_hash.py:38-43"""
    out = np.empty(p, dtype=np.float64)
    lib().orc_signs(_u64(sign_seed), p, _p(out))
    return out


def column_keys(master_seed: int, i0: int, i1: int, p: int) -> np.ndarray:
    """_hash.py:46-56"""
    out = np.empty((i1 - i0, p), dtype=np.uint64)
    lib().orc_column_keys(_u64(master_seed), i0, i1 - i0, p, _p(out))
    return out


def indices_block(master_seed: int, i0: int, i1: int, p: int, m: int) -> np.ndarray:
    """SamplingPlan.indices_block, sketch.py:48-56"""
    out = np.empty((i1 - i0, m), dtype=np.uint32)
    lib().orc_indices_block(_u64(master_seed), i0, i1 - i0, p, m, _p(out))
    return out


def philox4x32_10(ctr, key) -> np.ndarray:
    """One Philox4x32-10 block (Salmon et al. SC'11): 4 x u32 counter, 2 x u32 key."""
    c = np.array(ctr, dtype=np.uint32)
    lib().orc_philox4x32_10(_p(c), int(key[0]), int(key[1]))
    return c


def philox_indices(master_seed: int, i0: int, i1: int, p: int, m: int) -> np.ndarray:
    """The Philox sampler's kept sets (no reference counterpart; see sketch_oracle.c)."""
    out = np.empty((i1 - i0, m), dtype=np.uint32)
    lib().orc_philox_indices(_u64(master_seed), i0, i1 - i0, p, m, _p(out))
    return out


# ---- L1 transform (transform.py) -------------------------------------------------

def next_pow2(n: int) -> int:
    """transform.py:26-27"""
    return 1 << (int(n) - 1).bit_length()


def fwht(v: np.ndarray) -> np.ndarray:
    """_fwht_axis0 on one vector, transform.py:92-110 (returns a new array)."""
    a = np.array(v, dtype=np.float64, copy=True)
    lib().orc_fwht(_p(a), a.shape[0])
    return a


def precondition_rows(X: np.ndarray, p_pad: int, kind: int, sign_seed: int) -> np.ndarray:
    """precondition_columns on sample-major rows, transform.py:180-189"""
    X = np.ascontiguousarray(X, dtype=np.float64)
    n, p = X.shape
    Y = np.empty((n, p_pad), dtype=np.float64)
    lib().orc_precondition_rows(_p(X), p, n, p, p_pad, kind, _u64(sign_seed), _p(Y))
    return Y


def unprecondition_rows(Y: np.ndarray, kind: int, sign_seed: int) -> np.ndarray:
    """unprecondition_columns on sample-major rows, transform.py:192-200"""
    Y = np.ascontiguousarray(Y, dtype=np.float64)
    n, p_pad = Y.shape
    X = np.empty_like(Y)
    lib().orc_unprecondition_rows(_p(Y), n, p_pad, kind, _u64(sign_seed), _p(X))
    return X


# ---- L2 fused sketch (sketch.py:196-223) -------------------------------------------

def sketch(X: np.ndarray, p_pad: int, kind: int, sign_seed: int, master_seed: int, m: int,
           col0: int = 0, nthreads: int = 1):
    """sketch_stream on sample-major rows. X is fp32 or fp64 with shape (n, p).

    Returns indices (n, m) uint32 and values (n, m) float64.
    """
    if X.dtype == np.float32:
        X = np.ascontiguousarray(X)
        f32 = 1
    else:
        X = np.ascontiguousarray(X, dtype=np.float64)
        f32 = 0
    n, p = X.shape
    idx = np.empty((n, m), dtype=np.uint32)
    val = np.empty((n, m), dtype=np.float64)
    lib().orc_sketch(_p(X), f32, p, n, p, p_pad, kind, _u64(sign_seed), _u64(master_seed), col0, m,
                     _p(idx), _p(val), nthreads)
    return idx, val


# ---- L3a estimators (estimators.py) ----------------------------------------------

def mean_acc(idx: np.ndarray, val: np.ndarray, p_pad: int) -> np.ndarray:
    """bincount accumulation, estimators.py:39-43"""
    idx = np.ascontiguousarray(idx, dtype=np.uint32)
    val = np.ascontiguousarray(val, dtype=np.float64)
    acc = np.zeros(p_pad, dtype=np.float64)
    n, m = idx.shape
    lib().orc_mean_acc(_p(idx), _p(val), n, m, p_pad, _p(acc))
    return acc


def estimate_mean(idx, val, p: int, p_pad: int, kind: int, sign_seed: int) -> np.ndarray:
    """estimators.py:30-45"""
    n, m = idx.shape
    if n < 1:
        raise ValueError("empty sketch")
    acc = mean_acc(idx, val, p_pad)
    mean_pre = (p_pad / m) * acc / n
    return unprecondition_rows(mean_pre[None, :], kind, sign_seed)[0, :p]


def cov_acc(idx: np.ndarray, val: np.ndarray, p_pad: int, nthreads: int = 1) -> np.ndarray:
    """W @ W.T as a dense p_pad x p_pad matrix, estimators.py:60-61"""
    idx = np.ascontiguousarray(idx, dtype=np.uint32)
    val = np.ascontiguousarray(val, dtype=np.float64)
    n, m = idx.shape
    C = np.zeros((p_pad, p_pad), dtype=np.float64)
    lib().orc_cov_acc(_p(idx), _p(val), n, m, p_pad, _p(C), nthreads)
    return C


def cov_finalize(C: np.ndarray, p_pad: int, m: int, n: int) -> np.ndarray:
    """estimators.py:62-65 (scale, symmetrise, diagonal debias)"""
    C = C * ((p_pad * (p_pad - 1)) / (m * (m - 1)) / n)
    diag = C.diagonal().copy()
    C = 0.5 * (C + C.T)
    np.fill_diagonal(C, diag * (1.0 - (p_pad - m) / (p_pad - 1)))
    return C


def estimate_covariance(idx, val, p_pad: int, nthreads: int = 1) -> np.ndarray:
    """estimators.py:48-66"""
    n, m = idx.shape
    if m < 2:
        raise ValueError("covariance estimation needs m >= 2")
    if n < 1:
        raise ValueError("empty sketch")
    return cov_finalize(cov_acc(idx, val, p_pad, nthreads), p_pad, m, n)


def top_eigenvectors(C: np.ndarray, k: int) -> np.ndarray:
    """estimators.py:69-81 (LAPACK eigh, descending)"""
    w, V = np.linalg.eigh(0.5 * (C + C.T))
    return V[:, ::-1][:, :k]


def principal_components(idx, val, p: int, p_pad: int, kind: int, sign_seed: int, k: int) -> np.ndarray:
    """estimators.py:116-129"""
    V = top_eigenvectors(estimate_covariance(idx, val, p_pad), k)
    return unprecondition_rows(V.T, kind, sign_seed)[:, :p].T


# ---- L3b sparsified K-means (cluster.py) -------------------------------------------

def pairwise_sum(a: np.ndarray) -> float:
    """numpy pairwise summation, the order of ndarray.sum"""
    a = np.ascontiguousarray(a, dtype=np.float64)
    return float(lib().orc_pairwise_sum(_p(a), a.shape[0]))


def init_centers(idx, val, chosen, p_pad: int) -> np.ndarray:
    """_SparseOps.init_centers, cluster.py:175-179"""
    mu = np.zeros((p_pad, len(chosen)))
    for j, c in enumerate(chosen):
        mu[idx[c].astype(np.int64), j] = val[c]
    return mu


def kmeans_assign(idx, val, mu: np.ndarray, nthreads: int = 1):
    """_SparseOps.assign, cluster.py:181-187. Returns (labels int64, d2min f64)."""
    idx = np.ascontiguousarray(idx, dtype=np.uint32)
    val = np.ascontiguousarray(val, dtype=np.float64)
    mu = np.ascontiguousarray(mu, dtype=np.float64)
    n, m = idx.shape
    p, K = mu.shape
    labels = np.empty(n, dtype=np.int64)
    d2min = np.empty(n, dtype=np.float64)
    lib().orc_kmeans_assign(_p(idx), _p(val), n, m, _p(mu), p, K, _p(labels), _p(d2min), nthreads)
    return labels, d2min


def kmeans_update(idx, val, labels, mu_prev: np.ndarray):
    """_SparseOps.update, cluster.py:189-210. Returns (mu, counts int64, empty bool)."""
    idx = np.ascontiguousarray(idx, dtype=np.uint32)
    val = np.ascontiguousarray(val, dtype=np.float64)
    labels = np.ascontiguousarray(labels, dtype=np.int64)
    mu_prev = np.ascontiguousarray(mu_prev, dtype=np.float64)
    n, m = idx.shape
    p, K = mu_prev.shape
    mu = np.empty_like(mu_prev)
    counts = np.empty((p, K), dtype=np.int64)
    empty = np.empty(K, dtype=np.uint8)
    lib().orc_kmeans_update(_p(idx), _p(val), n, m, _p(labels), p, K, _p(mu_prev), _p(mu), _p(counts),
                            _p(empty))
    return mu, counts, empty.astype(bool)


def kmeans_reseed(idx, val, mu: np.ndarray, k: int, d2min: np.ndarray) -> None:
    """_SparseOps.reseed, cluster.py:212-215"""
    c = int(np.argmax(d2min))
    mu[:, k] = 0.0
    mu[idx[c].astype(np.int64), k] = val[c]


def lloyd(idx, val, mu0: np.ndarray, max_iter: int, nthreads: int = 1):
    """The Lloyd loop body of _lloyd_iterate, cluster.py:230-241, from given centers.

    Returns (labels, mu, objective trajectory, iterations).
    """
    mu = np.array(mu0, dtype=np.float64, copy=True)
    K = mu.shape[1]
    prev = None
    traj = []
    iters = 0
    labels = np.zeros(idx.shape[0], dtype=np.int64)
    for _ in range(max_iter):
        labels, d2min = kmeans_assign(idx, val, mu, nthreads)
        traj.append(float(d2min.sum()))
        iters += 1
        if prev is not None and np.array_equal(labels, prev):
            break
        prev = labels
        mu, _, empty = kmeans_update(idx, val, labels, mu)
        for k in np.flatnonzero(empty):
            kmeans_reseed(idx, val, mu, int(k), d2min)
    return labels, mu, traj, iters
