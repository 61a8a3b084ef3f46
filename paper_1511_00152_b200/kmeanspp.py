"""K-means++ seeding on the sketch; cluster.py:70-93 with _SparseOps.d2_to_point :169-173.

The D^2 vector to each new centre is computed on the device (``skc_kmeans_d2_to_point``,
fp64 in scipy's sparse-product order). The seeded D^2-weighted draws use numpy's PCG64
stream on the host, exactly as the reference does (``_restart_rng``, cluster.py:70-71).
Same seed gives the same centres.
"""

from __future__ import annotations

import numpy as np
import torch

from . import _lib
from .errors import ParameterError


def restart_rng(seed: int, restart: int) -> np.random.Generator:
    """cluster.py:70-71"""
    return np.random.default_rng([int(seed) & 0xFFFFFFFFFFFFFFFF, restart])


class _D2:
    def __init__(self, ops):
        self.ops = ops
        dev = ops.dev
        self.colsq = torch.empty(ops.n, dtype=torch.float64, device=dev)
        self.dense = torch.empty(ops.p, dtype=torch.float64, device=dev)
        self.out = torch.empty(ops.n, dtype=torch.float64, device=dev)
        with torch.cuda.device(dev):
            _lib.call("skc_row_sqnorms", ops.val.data_ptr(), ops.vcode, ops.n, ops.m, self.colsq.data_ptr(),
                      _lib.stream_ptr(dev))

    def __call__(self, c: int) -> np.ndarray:
        ops = self.ops
        with torch.cuda.device(ops.dev):
            _lib.call("skc_kmeans_d2_to_point", ops.idx.data_ptr(), ops.val.data_ptr(), ops.vcode, ops.n, ops.m,
                      ops.p, int(c), self.colsq.data_ptr(), self.dense.data_ptr(), self.out.data_ptr(),
                      _lib.stream_ptr(ops.dev))
        return self.out.cpu().numpy()


def pp_select(n: int, K: int, rng, d2_to_point) -> list:
    """D^2-weighted sequential seeding; cluster.py:74-93"""
    if K > n:
        raise ParameterError(f"K={K} exceeds number of points n={n}")
    if K < 1:
        raise ParameterError("K must be >= 1")
    chosen = [int(rng.integers(n))]
    if K == 1:
        return chosen
    d2 = d2_to_point(chosen[0])
    for _ in range(1, K):
        total = d2.sum()
        if total > 0:
            nxt = int(rng.choice(n, p=d2 / total))
        else:
            nxt = int(rng.integers(n))
        chosen.append(nxt)
        np.minimum(d2, d2_to_point(nxt), out=d2)
    return chosen


def kmeanspp_select(ops, K: int, seed: int, restart: int) -> list:
    """Chosen point indices of restart ``restart`` (cluster.py:224 via _best_of_restarts)."""
    return pp_select(ops.n, K, restart_rng(seed, restart), _D2(ops))
