"""Sample-dimension sharding over N GPUs (one process per GPU, torch.distributed/NCCL).

Each rank sketches the global columns [c0, c1) = shard_bounds(n, rank, world) with
``col0 = c0``. Signs, indices and values depend only on (x_i, global i, seeds)
(_hash.py:46-56), so a sharded sketch is byte-identical to the 1-GPU sketch. The
exchange steps are the reductions the reference spec allows:
  * estimators: ONE allreduce per pass of [mean acc (p), stats, packed triangle];
  * K-means: per Lloyd iteration, an allreduce of [changed, objective, d2max], a
    MIN-allreduce for the global first argmax, an allreduce of the K x p sums and
    counts, and a broadcast of the reseed row when a cluster empties.
All helpers reduce to no-ops when torch.distributed is not initialised or world == 1.
"""

from __future__ import annotations

from typing import Optional

import torch
import torch.distributed as dist


def world(group=None) -> int:
    return dist.get_world_size(group) if dist.is_available() and dist.is_initialized() else 1


def rank(group=None) -> int:
    return dist.get_rank(group) if dist.is_available() and dist.is_initialized() else 0


def shard_bounds(n: int, r: int, w: int) -> tuple[int, int]:
    """Contiguous, balanced column range of rank r out of w."""
    return (n * r) // w, (n * (r + 1)) // w


def owner_of(i: int, n: int, w: int) -> int:
    """Rank whose shard_bounds contain global column i."""
    r = (i * w) // n
    while shard_bounds(n, r, w)[0] > i:
        r -= 1
    while shard_bounds(n, r, w)[1] <= i:
        r += 1
    return r


def allreduce_(t: torch.Tensor, op=None, group=None) -> torch.Tensor:
    if world(group) > 1:
        dist.all_reduce(t, op=op or dist.ReduceOp.SUM, group=group)
    return t


def combine_moments(acc: torch.Tensor, stats: torch.Tensor, tri: Optional[torch.Tensor], n_local: int,
                    group=None) -> int:
    """Allreduce K2/K3 partials in place and return the global row count."""
    if world(group) == 1:
        return int(n_local)
    allreduce_(acc, group=group)
    mx = stats[1:2].clone()
    allreduce_(stats, group=group)  # sum of squares and rows add up
    allreduce_(mx, dist.ReduceOp.MAX, group=group)
    stats[1:2].copy_(mx)
    if tri is not None:
        allreduce_(tri, group=group)
    n = torch.tensor([int(n_local)], dtype=torch.int64, device=acc.device)
    allreduce_(n, group=group)
    return int(n.item())


def global_first_argmax(value: float, index: int, device, group=None) -> tuple[float, int]:
    """(max value, smallest global index attaining it) over ranks: np.argmax semantics."""
    if world(group) == 1:
        return value, index
    v = torch.tensor([value], dtype=torch.float64, device=device)
    allreduce_(v, dist.ReduceOp.MAX, group=group)
    key = torch.tensor([index if value == float(v.item()) and index >= 0 else 2**62], dtype=torch.int64,
                       device=device)
    allreduce_(key, dist.ReduceOp.MIN, group=group)
    return float(v.item()), int(key.item())


def broadcast_row(idx_row: Optional[torch.Tensor], val_row: Optional[torch.Tensor], m: int, val_dtype, owner: int,
                  device, group=None):
    """Send the reseed row (m indices + m values) from its owner rank to every rank."""
    if world(group) == 1:
        return idx_row, val_row
    i = idx_row.clone() if rank(group) == owner else torch.empty(m, dtype=torch.int32, device=device)
    v = val_row.clone() if rank(group) == owner else torch.empty(m, dtype=val_dtype, device=device)
    dist.broadcast(i, src=owner, group=group)
    dist.broadcast(v, src=owner, group=group)
    return i, v
