"""world_size-2 gloo tests of the sample-sharded path (no GPU needed).

Each rank sketches a contiguous column shard with its global offset (col0). Its partial
sums are computed by the CPU oracle, which stands in for the device kernels here. The
product's exchange logic then combines them: ``dist.combine_moments``, and
``cluster.lloyd_loop`` with its one packed allreduce per iteration (partials, changed count,
objective and every rank's (max d2min, global argmax) slot) and the reseed-row exchange.
The sharded results must equal the unsharded oracle run: sketch bytes and labels
exactly, sums to fp64 reduction-order tolerance.
"""

import os
import socket
import sys
import tempfile

import numpy as np
import pytest
import torch
import torch.distributed as tdist
import torch.multiprocessing as mp

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
WORLD = 2


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _data(p=64, n=3001, K=5, seed=7):
    rng = np.random.default_rng(seed)
    C = rng.standard_normal((p, K)) * 3.0
    X = (C[:, rng.integers(0, K, n)] + rng.standard_normal((p, n))).astype(np.float32)
    return X


class OracleShardOps:
    """The SketchKMeans interface of cluster.lloyd_loop, computed by the CPU oracle on one shard."""

    def __init__(self, idx, val, col0, p_pad):
        from oracle import oracle as O

        self.O = O
        self.idx_np, self.val_np = idx, val
        self.idx = torch.from_numpy(idx.astype(np.int32))
        self.val = torch.from_numpy(val)
        self.n, self.m = idx.shape
        self.p = p_pad
        self.col0 = col0
        self.dev = torch.device("cpu")

    def assign(self, mu, prev, labels, d2min, out, d2max):
        lab, d2 = self.O.kmeans_assign(self.idx_np, self.val_np, mu.numpy())
        labels.copy_(torch.from_numpy(lab.astype(np.int32)))
        d2min.copy_(torch.from_numpy(d2))
        out[0] = int((lab != prev.numpy()).sum()) if prev is not None else 0
        out[1] = int(np.argmax(d2)) if self.n else -1
        d2max[0] = float(d2.max()) if self.n else -1.0

    def objective(self, d2min, obj):
        obj[0] = self.O.pairwise_sum(d2min.numpy())

    def partials(self, labels, K):
        lab = labels.numpy().astype(np.int64)
        flat = self.idx_np.astype(np.int64) * K + lab[:, None]
        sums = torch.from_numpy(np.bincount(flat.ravel(), weights=self.val_np.ravel(), minlength=self.p * K)
                                .reshape(self.p, K))
        counts = torch.from_numpy(np.bincount(flat.ravel(), minlength=self.p * K).reshape(self.p, K))
        sizes = torch.from_numpy(np.bincount(lab, minlength=K).astype(np.int64))
        return sums, counts, sizes

    def centers(self, sums, counts, sizes, mu_prev):
        mu = mu_prev.clone()
        c = counts.to(torch.float64)
        upd = (counts > 0) & (sizes[None, :] > 0)
        mu[upd] = sums[upd] / c[upd]
        return mu, (sizes == 0).to(torch.int32)

    def reseed(self, mu, empty, idx_row, val_row):
        for k in torch.nonzero(empty).flatten().tolist():
            mu[:, k] = 0.0
            mu[idx_row.long(), k] = val_row.to(torch.float64)


def _worker(rank, world, port, outdir):
    sys.path.insert(0, ROOT)
    sys.path.insert(0, os.path.join(ROOT, "tests", "golden"))
    tdist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port}", rank=rank, world_size=world)
    from oracle import oracle as O
    from paper_1511_00152_b200 import dist
    from paper_1511_00152_b200.cluster import lloyd_loop

    X = _data()
    p, n = X.shape
    p_pad, m, ss, ms = 64, 12, 11, 12
    c0, c1 = dist.shard_bounds(n, rank, world)
    idx, val = O.sketch(X[:, c0:c1].T.copy(), p_pad, O.HADAMARD, ss, ms, m, col0=c0)
    # --- estimators: one allreduce of [acc, stats, packed triangle] per pass ---
    acc = torch.from_numpy(O.mean_acc(idx, val, p_pad))
    stats = torch.tensor([float((val * val).sum()), float(np.abs(val).max()), float(c1 - c0)], dtype=torch.float64)
    C = O.cov_acc(idx, val, p_pad)
    tri = torch.from_numpy(C[np.triu_indices(p_pad)].copy())
    n_tot = dist.combine_moments(acc, stats, tri, c1 - c0)
    # the same partials in one packed Moments buffer: exactly ONE collective for the pass
    from paper_1511_00152_b200.estimators import Moments

    calls = []
    real_allreduce = dist.allreduce_

    def counting_allreduce(t, op=None, group=None):
        calls.append(t.numel())
        return real_allreduce(t, op=op, group=group)

    dist.allreduce_ = counting_allreduce
    mom = Moments.zeros(p_pad, True, torch.device("cpu"))
    mom.acc.copy_(torch.from_numpy(O.mean_acc(idx, val, p_pad)))
    mom.stats.copy_(torch.tensor([float((val * val).sum()), float(np.abs(val).max()), float(c1 - c0)]))
    mom.tri.copy_(torch.from_numpy(C[np.triu_indices(p_pad)].copy()))
    n_packed = dist.combine_moments(mom.acc, mom.stats, mom.tri, c1 - c0)
    pass_calls = list(calls)
    # --- K-means: sharded Lloyd loop on UNEVEN shards (the reseed owner comes from every rank's
    # actual range); a duplicated start point forces an empty cluster ---
    K = 6
    idx_full, val_full = O.sketch(X.T.copy(), p_pad, O.HADAMARD, ss, ms, m)
    u0, u1 = (0, 1000) if rank == 0 else (1000, n)
    chosen = [5, 5, 100, 2000, 2999, 1500]
    mu0 = torch.from_numpy(O.init_centers(idx_full, val_full, chosen, p_pad))
    ops = OracleShardOps(idx_full[u0:u1], val_full[u0:u1], u0, p_pad)
    calls.clear()
    labels, mu, traj, iters, _ = lloyd_loop(ops, mu0, 30, None)
    loop_calls = list(calls)
    dist.allreduce_ = real_allreduce
    # --- sharded K-means++ host logic (kmeanspp._D2Sharded with the D^2 kernel in numpy):
    # owner's densified row + norm by one allreduce, D^2 shards by one all-gather ---
    from paper_1511_00152_b200.kmeanspp import pp_select, restart_rng

    sh_col0, sh_total = dist.shard_offset(u1 - u0)
    ranges = dist.shard_ranges(u0, u1 - u0, torch.device("cpu"))
    gathered = dist.gather_ranges(torch.arange(u0, u1, dtype=torch.float64), ranges)
    osum = dist.ordered_sum([0.1 * (rank + 1), 0.2 * (rank + 1)])
    li, lv = idx_full[u0:u1], val_full[u0:u1]
    colsq = (lv * lv).sum(axis=1)

    def d2_sharded(c):
        row = torch.zeros(p_pad + 1, dtype=torch.float64)
        if u0 <= c < u1:
            row[li[c - u0]] = torch.from_numpy(lv[c - u0])
            row[p_pad] = float(colsq[c - u0])
        dist.allreduce_(row)
        dense, csq = row[:p_pad].numpy(), float(row[p_pad])
        d2 = colsq + csq - 2.0 * (lv * dense[li]).sum(axis=1)
        return dist.gather_ranges(torch.from_numpy((p_pad / m) * np.clip(d2, 0.0, None)), ranges)

    pp = pp_select(sh_total, 6, restart_rng(3, 1), d2_sharded)
    np.savez(os.path.join(outdir, f"r{rank}.npz"), idx=idx, val=val, acc=acc.numpy(), stats=stats.numpy(),
             tri=tri.numpy(), n_tot=n_tot, labels=labels.numpy(), mu=mu.numpy(), traj=np.array(traj), iters=iters,
             packed=mom.packed.numpy(), n_packed=n_packed, pass_calls=np.array(pass_calls),
             loop_calls=np.array(loop_calls), shard=np.array([u0, u1]), sh=np.array([sh_col0, sh_total]),
             gathered=gathered, osum=osum, pp=np.array(pp))
    tdist.barrier()
    tdist.destroy_process_group()


@pytest.fixture(scope="module")
def sharded():
    with tempfile.TemporaryDirectory() as d:
        mp.spawn(_worker, args=(WORLD, _free_port(), d), nprocs=WORLD, join=True)
        yield [dict(np.load(os.path.join(d, f"r{r}.npz"))) for r in range(WORLD)]


def test_sharded_sketch_is_byte_identical(sharded):
    from oracle import oracle as O

    X = _data()
    idx, val = O.sketch(X.T.copy(), 64, O.HADAMARD, 11, 12, 12)
    assert np.array_equal(np.concatenate([r["idx"] for r in sharded]), idx)
    assert np.array_equal(np.concatenate([r["val"] for r in sharded]), val)


def test_combined_moments_equal_unsharded(sharded):
    from oracle import oracle as O

    X = _data()
    idx, val = O.sketch(X.T.copy(), 64, O.HADAMARD, 11, 12, 12)
    for r in sharded:
        assert int(r["n_tot"]) == X.shape[1]
        assert np.allclose(r["acc"], O.mean_acc(idx, val, 64), rtol=1e-12, atol=1e-12)
        assert np.allclose(r["tri"], O.cov_acc(idx, val, 64)[np.triu_indices(64)], rtol=1e-12, atol=1e-10)
        # max |v| is summed with the rest (one packed allreduce): an upper bound of the global max
        assert np.abs(val).max() <= r["stats"][1] <= WORLD * np.abs(val).max()
        assert np.isclose(r["stats"][0], (val * val).sum(), rtol=1e-12)
    assert np.array_equal(sharded[0]["tri"], sharded[1]["tri"])  # every rank holds the same result


def test_sharded_lloyd_matches_single_process(sharded):
    from oracle import oracle as O

    X = _data()
    idx, val = O.sketch(X.T.copy(), 64, O.HADAMARD, 11, 12, 12)
    mu0 = O.init_centers(idx, val, [5, 5, 100, 2000, 2999, 1500], 64)
    labels, mu, traj, iters = O.lloyd(idx, val, mu0, 30)
    got = np.concatenate([r["labels"] for r in sharded])
    assert int(sharded[0]["iters"]) == iters == int(sharded[1]["iters"])
    assert np.array_equal(got, labels)
    assert np.allclose(sharded[0]["traj"], traj, rtol=1e-12)
    assert np.allclose(sharded[0]["mu"], mu, rtol=1e-12, atol=1e-12)
    assert np.array_equal(sharded[0]["mu"], sharded[1]["mu"])


def test_one_collective_per_pass_and_per_iteration(sharded):
    """SPEC.md:212/:352 combine: the packed moments take ONE allreduce per pass; the Lloyd loop
    takes ONE per iteration (the packed exchange), plus one per iteration that empties a
    cluster (the reseed row), plus one at the start (every rank's range)."""
    for r in sharded:
        assert list(r["pass_calls"]) == [64 + 3 + 64 * 65 // 2]
        assert np.allclose(r["packed"][:64], sharded[0]["acc"], rtol=1e-12, atol=1e-12)
        assert int(r["n_packed"]) == int(r["n_tot"])
        calls = list(r["loop_calls"])
        it = int(r["iters"])
        exchange = 2 * 64 * 6 + 6 + 2 + 2 * 2  # sums, counts, sizes, changed, objective, 2 rank slots
        assert calls[0] == 4  # shard_ranges: (col0, n) of the 2 ranks
        assert calls.count(exchange) == it
        reseeds = [c for c in calls[1:] if c != exchange]
        assert all(c == 2 * 12 for c in reseeds) and len(reseeds) >= 1  # the forced empty cluster


def test_uneven_shards_lloyd_matches_single_process(sharded):
    from oracle import oracle as O

    X = _data()
    idx, val = O.sketch(X.T.copy(), 64, O.HADAMARD, 11, 12, 12)
    mu0 = O.init_centers(idx, val, [5, 5, 100, 2000, 2999, 1500], 64)
    lo, muo, to, io = O.lloyd(idx, val, mu0, 30)
    labels = np.concatenate([r["labels"] for r in sharded])
    assert [tuple(r["shard"]) for r in sharded] == [(0, 1000), (1000, 3001)]
    assert np.array_equal(labels, lo) and int(sharded[0]["iters"]) == io
    assert np.allclose(sharded[0]["mu"], muo, rtol=1e-12, atol=1e-12)


def test_shard_offsets_gather_and_ordered_sum(sharded):
    n = _data().shape[1]
    assert [tuple(r["sh"]) for r in sharded] == [(0, n), (1000, n)]
    for r in sharded:
        assert np.array_equal(r["gathered"], np.arange(n, dtype=np.float64))
        assert float(r["osum"]) == ((0.0 + 0.1) + 0.2) + 0.2 + 0.4  # rank order, then list order


def test_sharded_kmeanspp_chooses_the_unsharded_points(sharded):
    """cluster.py:74-93 on a sharded sketch: every rank draws from the global D^2 vector."""
    from oracle import oracle as O
    from paper_1511_00152_b200.kmeanspp import pp_select, restart_rng

    X = _data()
    idx, val = O.sketch(X.T.copy(), 64, O.HADAMARD, 11, 12, 12)
    colsq = (val * val).sum(axis=1)

    def d2_full(c):
        dense = np.zeros(64)
        dense[idx[c]] = val[c]
        d2 = colsq + colsq[c] - 2.0 * (val * dense[idx]).sum(axis=1)
        return (64 / 12) * np.clip(d2, 0.0, None)

    want = pp_select(X.shape[1], 6, restart_rng(3, 1), d2_full)
    for r in sharded:
        assert list(r["pp"]) == want
