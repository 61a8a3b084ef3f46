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


class _D2Sharded(_D2):
    """D^2 to a GLOBAL point over a sample-sharded sketch (rank r holds [col0, col0 + n)).

    The owner of point c puts W[:, c] densified and colsq[c] in a (p_pad + 1) buffer, one
    SUM allreduce hands it to every rank, each rank runs ``skc_kmeans_d2_to_dense`` on its
    shard (the arithmetic of d2_to_point), and one all-gather assembles the global vector.
    Every rank then makes the same host draws, so the chosen points equal the unsharded ones."""

    def __init__(self, ops, group=None):
        super().__init__(ops)
        from . import dist

        self.dist, self.group = dist, group
        self.ranges = dist.shard_ranges(int(ops.col0), ops.n, ops.dev, group)
        self.n_total = sum(n for _, n in self.ranges)
        self.row = torch.empty(ops.p + 1, dtype=torch.float64, device=ops.dev)

    def __call__(self, c: int) -> np.ndarray:
        ops, c0 = self.ops, int(self.ops.col0)
        self.row.zero_()
        if c0 <= c < c0 + ops.n:
            self.row[: ops.p] = ops.init_centers(np.array([c - c0], dtype=np.int64))[:, 0]
            self.row[ops.p] = self.colsq[c - c0]
        self.dist.allreduce_(self.row, group=self.group)
        with torch.cuda.device(ops.dev):
            _lib.call("skc_kmeans_d2_to_dense", ops.idx.data_ptr(), ops.val.data_ptr(), ops.vcode, ops.n, ops.m,
                      ops.p, self.row.data_ptr(), self.row[ops.p:].data_ptr(), self.colsq.data_ptr(),
                      self.out.data_ptr(), _lib.stream_ptr(ops.dev))
        return self.dist.gather_ranges(self.out, self.ranges, self.group)


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


def kmeanspp_select(ops, K: int, seed: int, restart: int, group=None) -> list:
    """Chosen point indices of restart ``restart`` (cluster.py:224 via _best_of_restarts).

    Under torch.distributed (world > 1) ``ops`` holds one shard and the indices are global."""
    from . import dist

    if dist.world(group) > 1:
        d2 = _D2Sharded(ops, group)
        return pp_select(d2.n_total, K, restart_rng(seed, restart), d2)
    return pp_select(ops.n, K, restart_rng(seed, restart), _D2(ops))
