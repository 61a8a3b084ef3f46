"""Sample-dimension sharding over N GPUs (one process per GPU, torch.distributed/NCCL).

Each rank sketches the global columns [c0, c1) = shard_bounds(n, rank, world) with
``col0 = c0``. Signs, indices and values depend only on (x_i, global i, seeds)
(_hash.py:46-56), so a sharded sketch is byte-identical to the 1-GPU sketch. The
exchange steps are the reductions the reference spec allows:
  * estimators: ONE allreduce per pass of [mean acc (p), stats, packed triangle];
  * K-means: per Lloyd iteration ONE allreduce of the packed exchange [sums | counts |
    sizes | changed | objective | per-rank (max d2min, argmax row)] (cluster.py
    _lloyd_loop_sharded), plus one of the reseed row when a cluster empties;
  * K-means++ seeding: per chosen point, one allreduce of its densified row and norm and
    one all-gather of the D^2 shards, so every rank draws from the global D^2 vector.
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


def _packed_span(acc: torch.Tensor, stats: torch.Tensor, tri: Optional[torch.Tensor]) -> Optional[torch.Tensor]:
    """The one contiguous fp64 buffer [acc | stats | tri] the three are views of, if they are."""
    if not (acc.is_contiguous() and stats.is_contiguous() and acc.dtype == stats.dtype == torch.float64):
        return None
    p = acc.numel()
    if stats.data_ptr() != acc.data_ptr() + 8 * p or stats.numel() != 3:
        return None
    total = p + 3
    if tri is not None:
        if not tri.is_contiguous() or tri.dtype != torch.float64 or tri.data_ptr() != stats.data_ptr() + 24:
            return None
        total += tri.numel()
    return torch.as_strided(acc, (total,), (1,))


def combine_moments(acc: torch.Tensor, stats: torch.Tensor, tri: Optional[torch.Tensor], n_local: int,
                    group=None, n_total: Optional[int] = None) -> int:
    """Sum the K2/K3 partials of every rank in place with ONE allreduce; return the global rows.

    acc / stats / tri are views of Moments.packed (one buffer), so the exchange is a single
    fp64 SUM allreduce of [acc | stats | tri] (4.2 MB at p=1024). stats[1] (max |v|) is
    summed too: the sum of the ranks' maxima bounds the global maximum, which is all a later
    K3t scale needs; finalize does not read it. The global row count is stats[2] after the
    sum; pass ``n_total`` when the caller knows it to avoid a device read.
    """
    if world(group) == 1:
        return int(n_local)
    buf = _packed_span(acc, stats, tri)
    if buf is not None:
        allreduce_(buf, group=group)
    else:  # separately allocated partials: pack, one allreduce, unpack
        parts = [acc.reshape(-1), stats.reshape(-1)] + ([tri.reshape(-1)] if tri is not None else [])
        buf = torch.cat(parts)
        allreduce_(buf, group=group)
        o = 0
        for t in parts:
            t.copy_(buf[o:o + t.numel()])
            o += t.numel()
    if n_total is not None:
        return int(n_total)
    return int(round(float(stats[2].item())))


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


def init_centers_global(ops, chosen) -> torch.Tensor:
    """init_centers (cluster.py:175-179) from GLOBAL point indices over sharded ops: each rank
    fills the centres whose point lies in its shard [ops.col0, ops.col0 + ops.n), the others
    stay zero, and one SUM allreduce gives every rank the full (p_pad, K) matrix."""
    import numpy as np

    chosen = np.asarray(chosen, dtype=np.int64)
    if world() == 1 and int(getattr(ops, "col0", 0)) == 0:
        return ops.init_centers(chosen)
    c0, n = int(ops.col0), int(ops.n)
    K = int(chosen.shape[0])
    mu = torch.zeros((ops.p, K), dtype=torch.float64, device=ops.dev)
    mine = np.flatnonzero((chosen >= c0) & (chosen < c0 + n))
    if mine.size:
        mu[:, torch.as_tensor(mine, device=ops.dev)] = ops.init_centers(chosen[mine] - c0)
    return allreduce_(mu)


def shard_ranges(col0: int, n: int, device, group=None) -> list:
    """Every rank's global column range [(col0, n)], from one allreduce (ranks may be uneven)."""
    w = world(group)
    if w == 1:
        return [(int(col0), int(n))]
    t = torch.zeros((w, 2), dtype=torch.int64, device=device)
    t[rank(group), 0] = int(col0)
    t[rank(group), 1] = int(n)
    allreduce_(t, group=group)
    return [(int(a), int(b)) for a, b in t.cpu().tolist()]


def collective_device():
    """Device for small host-logic collectives: the current CUDA device under NCCL, else CPU."""
    if world() > 1 and dist.get_backend() == "nccl":
        return torch.device("cuda", torch.cuda.current_device())
    return torch.device("cpu")


def shard_offset(n_local: int, group=None) -> tuple[int, int]:
    """(col0, n_total) of this rank when shards are concatenated in rank order."""
    w = world(group)
    if w == 1:
        return 0, int(n_local)
    t = torch.zeros(w, dtype=torch.int64, device=collective_device())
    t[rank(group)] = int(n_local)
    allreduce_(t, group=group)
    sizes = t.cpu().tolist()
    return int(sum(sizes[: rank(group)])), int(sum(sizes))


def gather_ranges(local: torch.Tensor, ranges: list, group=None):
    """Concatenate every rank's 1-D shard ``local`` into the global host (numpy) vector.

    ``ranges`` is shard_ranges' [(col0, n)] per rank; together they must tile [0, total).
    One all-gather of max(n)-padded buffers."""
    import numpy as np

    total = sum(n for _, n in ranges)
    if world(group) == 1:
        return local.cpu().numpy()
    nmax = max(max(n for _, n in ranges), 1)
    on = torch.device("cpu") if dist.get_backend(group) == "gloo" else local.device
    buf = torch.zeros(nmax, dtype=local.dtype, device=on)
    buf[: local.numel()] = local
    parts = [torch.empty_like(buf) for _ in ranges]
    dist.all_gather(parts, buf, group=group)
    out = np.empty(total, dtype=buf.cpu().numpy().dtype)
    covered = 0
    for (c0, n), part in zip(ranges, parts):
        if c0 < 0 or c0 + n > total:
            raise ValueError("shard ranges do not tile [0, total)")
        out[c0:c0 + n] = part[:n].cpu().numpy()
        covered += n
    if covered != total:
        raise ValueError("shard ranges do not tile [0, total)")
    return out


def ordered_sum(values: list, group=None) -> float:
    """Sum every rank's list of floats in (rank, position) order, as one process would."""
    if world(group) == 1:
        allv = [values]
    else:
        allv = [None] * world(group)
        dist.all_gather_object(allv, [float(v) for v in values], group=group)
    tot = 0.0
    for vs in allv:
        for v in vs:
            tot += float(v)
    return tot
