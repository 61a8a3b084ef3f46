"""Sample-sharded path on the real CUDA kernels: 2 processes sharing the one GPU over gloo.

Each rank sketches its global column shard (col0) with the product kernels, accumulates its
moments, and runs the sharded Lloyd loop (one packed allreduce per iteration, packed by
skc_kmeans_pack_exchange). The ranks never wait on each other inside a kernel: gloo moves the
buffers through the host between launches. Against the unsharded run in this process:
  sketch indices and fp64 values   bit-identical (global column offsets, _hash.py:46-56)
  covariance / mean partials       equal to fp64 summation-order tolerance
  labels, counts, iterations       identical; centres and objective to summation order
Also: the NCCL entry points of the C ABI on a 1-rank communicator.
"""

import ctypes
import os
import socket
import sys
import tempfile

import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
WORLD = 2
P, N, M, K = 256, 30001, 25, 6
SS, MS = 11, 12
CHOSEN = [5, 5, 100, 20000, 29999, 15000]  # a duplicated start point empties a cluster


def _port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _data():
    rng = np.random.default_rng(7)
    C = rng.standard_normal((P, K)) * 3.0
    return (C[:, rng.integers(0, K, N)] + rng.standard_normal((P, N))).T.astype(np.float32).copy()  # (n, p)


def _run(skc, X, col0, n_total):
    from paper_1511_00152_b200 import dist

    dev = torch.device("cuda", 0)
    spec = skc.PreconditionSpec.create("hadamard", P, sign_seed=SS)
    plan = skc.SamplingPlan(MS, P, M)
    sk = skc.sketch_stream(skc.RowSource(torch.as_tensor(X, device=dev)), spec, plan, col0=col0)
    mom = skc.accumulate_moments(sk)
    dist.combine_moments(mom.acc, mom.stats, mom.tri, sk.n, n_total=n_total)
    ops = skc.SketchKMeans(sk)
    mu0 = dist.init_centers_global(ops, CHOSEN)
    labels, mu, traj, iters, _ = ops.lloyd(mu0, 30)
    counts = dist.allreduce_(ops.partials(labels, K)[1])  # per-(coordinate, cluster) sampling counts
    # the public API on the shard: K-means++ restarts (sharded D^2 draws), then the two-pass variant
    Xd = torch.as_tensor(X, device=dev)
    res = skc.sparsified_kmeans(skc.RowSource(Xd), K, M / P, max_iter=30, n_init=2, seed=5)
    res2 = skc.sparsified_kmeans_two_pass(skc.RowSource(Xd, chunk_cols=4096), K, M / P, max_iter=30, n_init=1,
                                          seed=5)
    return dict(idx=sk.host_indices(), val=sk.host_values(), acc=mom.acc.cpu().numpy(), tri=mom.tri.cpu().numpy(),
                labels=labels.cpu().numpy(), mu=mu.cpu().numpy(), traj=np.array(traj), iters=iters,
                counts=counts.cpu().numpy(), api_labels=res.assignments.labels, api_obj=res.objective,
                api_centers=res.centers.centers, api_curve=np.array(res.diagnostics["objective_curve"]),
                tp_labels=res2.assignments.labels, tp_obj=res2.objective, tp_centers=res2.centers.centers)


def _worker(rank, world, port, outdir):
    sys.path.insert(0, ROOT)
    import torch.distributed as tdist

    torch.cuda.set_device(0)
    tdist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port}", rank=rank, world_size=world)
    import paper_1511_00152_b200 as skc
    from paper_1511_00152_b200 import dist

    X = _data()
    c0, c1 = dist.shard_bounds(N, rank, world)
    r = _run(skc, X[c0:c1], c0, N)
    np.savez(os.path.join(outdir, f"r{rank}.npz"), **r)
    tdist.barrier()
    tdist.destroy_process_group()


@pytest.fixture(scope="module")
def runs():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import torch.multiprocessing as mp

    import paper_1511_00152_b200 as skc

    with tempfile.TemporaryDirectory() as d:
        mp.spawn(_worker, args=(WORLD, _port(), d), nprocs=WORLD, join=True)
        shards = [dict(np.load(os.path.join(d, f"r{r}.npz"), allow_pickle=False)) for r in range(WORLD)]
    full = _run(skc, _data(), 0, N)
    return shards, full


def test_sharded_sketch_bit_identical(runs):
    shards, full = runs
    assert np.array_equal(np.concatenate([s["idx"] for s in shards]), full["idx"])
    assert np.array_equal(np.concatenate([s["val"] for s in shards]), full["val"])


def test_sharded_moments_one_allreduce(runs):
    shards, full = runs
    for s in shards:
        assert np.allclose(s["acc"], full["acc"], rtol=1e-12, atol=1e-12)
        assert np.abs(s["tri"] - full["tri"]).max() <= 1e-12 * np.abs(full["tri"]).max()
    assert np.array_equal(shards[0]["tri"], shards[1]["tri"])  # every rank holds the same result


def test_sharded_lloyd_matches_unsharded(runs):
    shards, full = runs
    assert all(int(s["iters"]) == full["iters"] for s in shards)
    assert np.array_equal(np.concatenate([s["labels"] for s in shards]), full["labels"])
    for s in shards:
        assert np.array_equal(s["counts"], full["counts"])
        assert np.abs(s["mu"] - full["mu"]).max() <= 1e-12 * np.abs(full["mu"]).max()
        assert np.allclose(s["traj"], full["traj"], rtol=1e-12)
    assert np.array_equal(shards[0]["mu"], shards[1]["mu"])


def test_sharded_public_kmeans_matches_unsharded(runs):
    """sparsified_kmeans on shards (col0 from rank order, K-means++ restarts drawn from the
    global D^2 vector) equals the one-process run: same seeds, same labels and trajectory."""
    shards, full = runs
    assert np.array_equal(np.concatenate([s["api_labels"] for s in shards]), full["api_labels"])
    for s in shards:
        assert len(s["api_curve"]) == len(full["api_curve"])
        assert np.allclose(s["api_curve"], full["api_curve"], rtol=1e-12)
        assert np.abs(s["api_centers"] - full["api_centers"]).max() <= 1e-12 * np.abs(full["api_centers"]).max()
    assert np.array_equal(shards[0]["api_centers"], shards[1]["api_centers"])


def test_sharded_two_pass_matches_unsharded(runs):
    shards, full = runs
    assert np.array_equal(np.concatenate([s["tp_labels"] for s in shards]), full["tp_labels"])
    for s in shards:
        assert np.isclose(float(s["tp_obj"]), float(full["tp_obj"]), rtol=1e-12)
        assert np.abs(s["tp_centers"] - full["tp_centers"]).max() <= 1e-12 * np.abs(full["tp_centers"]).max()


def test_d2_to_dense_equals_d2_to_point():
    """skc_kmeans_d2_to_dense with the point's own densified row == skc_kmeans_d2_to_point."""
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_1511_00152_b200 as skc
    from paper_1511_00152_b200 import _lib
    from paper_1511_00152_b200.kmeanspp import _D2

    dev = torch.device("cuda", 0)
    X = _data()[:5000]
    spec = skc.PreconditionSpec.create("hadamard", P, sign_seed=SS)
    sk = skc.sketch_stream(skc.RowSource(torch.as_tensor(X, device=dev)), spec, skc.SamplingPlan(MS, P, M))
    ops = skc.SketchKMeans(sk)
    d2 = _D2(ops)
    for c in (0, 1234, 4999):
        want = d2(c)
        row = torch.zeros(P + 1, dtype=torch.float64, device=dev)
        row[:P] = ops.init_centers(np.array([c]))[:, 0]
        row[P] = d2.colsq[c]
        out = torch.empty(ops.n, dtype=torch.float64, device=dev)
        _lib.call("skc_kmeans_d2_to_dense", ops.idx.data_ptr(), ops.val.data_ptr(), ops.vcode, ops.n, ops.m, P,
                  row.data_ptr(), row[P:].data_ptr(), d2.colsq.data_ptr(), out.data_ptr(), _lib.stream_ptr(dev))
        assert np.array_equal(out.cpu().numpy(), want)


def test_nccl_entry_points_single_rank():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_1511_00152_b200 import _lib
    from paper_1511_00152_b200.errors import ParameterError

    L = _lib.lib()
    torch.cuda.set_device(0)
    uid = ctypes.create_string_buffer(128)
    _lib.call("skc_nccl_get_unique_id", ctypes.addressof(uid))
    comm = ctypes.c_void_p()
    _lib.call("skc_nccl_comm_init_rank", ctypes.addressof(comm), 1, ctypes.addressof(uid), 0)
    try:
        p, K_, w = 64, 5, 1
        n_ex = L.skc_kmeans_exchange_len(p, K_, w)
        assert n_ex == 2 * p * K_ + K_ + 2 + 2 * w
        dev = torch.device("cuda", 0)
        sums = torch.randn((p, K_), dtype=torch.float64, device=dev)
        counts = torch.randint(0, 1000, (p, K_), dtype=torch.int64, device=dev)
        sizes = torch.randint(0, 1000, (K_,), dtype=torch.int64, device=dev)
        out = torch.tensor([17, 3], dtype=torch.int64, device=dev)
        d2max = torch.tensor([2.5], dtype=torch.float64, device=dev)
        obj = torch.tensor([123.25], dtype=torch.float64, device=dev)
        buf = torch.full((n_ex,), np.nan, dtype=torch.float64, device=dev)
        st = _lib.stream_ptr(dev)
        _lib.call("skc_kmeans_pack_exchange", sums.data_ptr(), counts.data_ptr(), sizes.data_ptr(), out.data_ptr(),
                  d2max.data_ptr(), obj.data_ptr(), p, K_, 0, w, 1000, buf.data_ptr(), st)
        _lib.call("skc_allreduce_sum_f64", buf.data_ptr(), n_ex, comm.value, st)  # one rank: identity
        s2, c2, z2 = torch.empty_like(sums), torch.empty_like(counts), torch.empty_like(sizes)
        _lib.call("skc_kmeans_unpack_exchange", buf.data_ptr(), p, K_, s2.data_ptr(), c2.data_ptr(), z2.data_ptr(), st)
        torch.cuda.synchronize()
        assert torch.equal(s2, sums) and torch.equal(c2, counts) and torch.equal(z2, sizes)
        tail = buf[2 * p * K_ + K_:].cpu().tolist()
        assert tail == [17.0, 123.25, 2.5, 1003.0]
        assert L.skc_moments_packed_len(256, 1) == 256 + 3 + 256 * 257 // 2
        with pytest.raises(ParameterError):
            _lib.call("skc_allreduce_sum_f64", buf.data_ptr(), n_ex, None, st)
    finally:
        _lib.call("skc_nccl_comm_destroy", comm.value)
