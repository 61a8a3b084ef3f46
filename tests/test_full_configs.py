"""Parity at every BASELINE.json config's stated n (C1-C5), on the bench's own generators.

The oracle (oracle/, pinned bit for bit to the reference's golden fixtures by
test_oracle_golden.py) runs the whole job on the host's cores in chunks of rows, with the
global column offset, so a chunk's sketch equals the full job's rows (sketch.py:196-223,
tests/test_sketch.py:161-171 chunk invariance).

  C1 p=256   n=20,000      sketch bit-exact, mean 1e-12, covariance 1e-6, top-5 PCs (up to sign)
  C2 p=512   n=200,000     Lloyd (K=10, <=20 iterations, seeded points): labels, objective
                           trajectory, centres and counts bit-exact
  C3 p=1024  n=2^24        f64 sketch bit-exact in every chunk; covariance <= 1e-5 relative
                           Frobenius in f64 and f32 compute (the north_star bound)
  C4 p=4096  n=2^21        the same, plus the top-20 eigenvector subspace
  C5 p=2048  n=10^7        every Lloyd iteration: labels and d2min of 10^5 sampled points
                           against the oracle's assignment with the device centres; counts and
                           centres of the whole job at the first and last update
"""

import os

import numpy as np
import pytest
import torch

from oracle import oracle as O

pytestmark = pytest.mark.gpu

SEED = 2026
NT = os.cpu_count() or 1


@pytest.fixture(scope="module")
def env():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import bench
    import paper_1511_00152_b200 as skc

    return skc, bench


def rel_fro(a, b):
    return float(np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-300))


def spec_plan(skc, bench, wl):
    c = bench.WORKLOADS[wl]
    spec = skc.PreconditionSpec.create("hadamard", c["p"], sign_seed=bench.derive_seed(SEED, 0xD5))
    plan = skc.SamplingPlan(bench.derive_seed(SEED, 0x5A), spec.p_pad, c["m"])
    return c, spec, plan


def test_c1_full(env):
    skc, bench = env
    c, spec, plan = spec_plan(skc, bench, "c1")
    n, p, m = c["n"], c["p"], c["m"]
    X = bench.gen_rows("c1", n, 0, torch.device("cuda"), torch)
    Xh = X.cpu().numpy()
    sk = skc.sketch_stream(skc.RowSource(X), spec, plan)  # drop-in default: compute f64
    io, vo = O.sketch(Xh, p, O.HADAMARD, spec.sign_seed, plan.master_seed, m, nthreads=NT)
    assert np.array_equal(sk.host_indices(), io) and np.array_equal(sk.host_values(), vo)
    mean = skc.estimate_mean(sk)
    mo = O.estimate_mean(io, vo, p, p, O.HADAMARD, spec.sign_seed)
    assert np.abs(mean - mo).max() <= 1e-12 * np.abs(mo).max()
    C = skc.estimate_covariance(sk).matrix
    Co = O.estimate_covariance(io, vo, p, nthreads=NT)
    err = rel_fro(C, Co)
    print(f"C1 covariance rel Frobenius error {err:.3e}")
    assert err < 1e-6
    U = skc.principal_components(sk, 5)
    Uo = O.unprecondition_rows(O.top_eigenvectors(Co, 5).T, O.HADAMARD, spec.sign_seed)[:, :p].T
    sgn = np.sign(np.sum(U * Uo, axis=0))
    assert np.abs(U * sgn - Uo).max() < 1e-6


def test_c2_full_lloyd(env):
    skc, bench = env
    c, spec, plan = spec_plan(skc, bench, "c2")
    n, p, m, K = c["n"], c["p"], c["m"], c["K"]
    X = bench.gen_rows("c2", n, 0, torch.device("cuda"), torch)
    sk = skc.sketch_stream(skc.RowSource(X), spec, plan)
    io, vo = O.sketch(X.cpu().numpy(), p, O.HADAMARD, spec.sign_seed, plan.master_seed, m, nthreads=NT)
    assert np.array_equal(sk.host_indices(), io) and np.array_equal(sk.host_values(), vo)
    chosen = np.random.default_rng(SEED).choice(n, K, replace=False)
    ops = skc.SketchKMeans(sk)
    labels, mu, traj, iters, _ = ops.lloyd(ops.init_centers(chosen), c["iters"])
    lo, muo, to, it_o = O.lloyd(io, vo, O.init_centers(io, vo, chosen, p), c["iters"], nthreads=NT)
    print(f"C2 Lloyd: {iters} iterations, objective {traj[-1]!r}")
    assert iters == it_o and traj == to
    assert np.array_equal(labels.cpu().numpy(), lo)
    assert np.array_equal(mu.cpu().numpy(), muo)
    _, counts, _ = ops.update(labels, mu)
    _, co, _ = O.kmeans_update(io, vo, lo, muo)
    assert np.array_equal(counts.cpu().numpy(), co)


def _streamed_covariance(skc, bench, wl, chunk, pcs=0):
    c, spec, plan = spec_plan(skc, bench, wl)
    n, p, m = c["n"], c["p"], c["m"]
    dev = torch.device("cuda")
    moms = {"f64": None, "f32": None}
    Cacc = np.zeros((p, p))
    for r0 in range(0, n, chunk):
        X = bench.gen_rows(wl, chunk, r0, dev, torch)
        src = skc.RowSource(X)
        for comp in moms:
            moms[comp] = skc.stream_moments(src, spec, plan, compute=comp, col0=r0, into=moms[comp])
        sk = skc.sketch_stream(src, spec, plan, compute="f64", col0=r0)
        io, vo = O.sketch(X.cpu().numpy(), p, O.HADAMARD, spec.sign_seed, plan.master_seed, m, col0=r0, nthreads=NT)
        assert np.array_equal(sk.host_indices(), io), f"indices differ in chunk {r0}"
        assert np.array_equal(sk.host_values(), vo), f"fp64 values differ in chunk {r0}"
        Cacc += O.cov_acc(io, vo, p, nthreads=NT)
        del X, sk, src
    Co = O.cov_finalize(Cacc, p, m, n)
    out = {}
    for comp, mom in moms.items():
        C = skc.covariance_from_moments(mom, p, m, n).cpu().numpy()
        out[comp] = (C, rel_fro(C, Co))
        print(f"{wl.upper()} n={n} compute={comp}: covariance rel Frobenius error {out[comp][1]:.3e}")
    torch.cuda.empty_cache()
    return Co, out


def test_c3_full_covariance(env):
    skc, bench = env
    _, out = _streamed_covariance(skc, bench, "c3", 1 << 20)
    assert out["f64"][1] < 1e-5 and out["f32"][1] < 1e-5


def test_c4_full_covariance_and_pcs(env):
    skc, bench = env
    Co, out = _streamed_covariance(skc, bench, "c4", 1 << 18)
    assert out["f64"][1] < 1e-5 and out["f32"][1] < 1e-5
    k = 20
    V = skc.top_eigenvectors(out["f64"][0], k)
    Vo = O.top_eigenvectors(Co, k)
    # subspace distance: sine of the largest principal angle (robust to rotations inside
    # clusters of near-equal eigenvalues); eigenvector signs are parity-unpinned
    s = np.linalg.svd(Vo.T @ V, compute_uv=False)
    sin_max = float(np.sqrt(max(0.0, 1.0 - s.min() ** 2)))
    print(f"C4 top-{k} subspace: sin(max principal angle) {sin_max:.3e}")
    assert sin_max < 1e-5


def test_c5_full_lloyd_sampled(env):
    skc, bench = env
    c, spec, plan = spec_plan(skc, bench, "c5")
    n, p, m, K = c["n"], c["p"], c["m"], c["K"]
    dev = torch.device("cuda")
    X = bench.gen_rows("c5", n, 0, dev, torch)
    sk = skc.sketch_stream(skc.RowSource(X), spec, plan)
    # a sample of rows: the sketch itself against the oracle
    rng = np.random.default_rng(5)
    S = np.sort(rng.choice(n, 100_000, replace=False))
    St = torch.as_tensor(S, device=dev)
    Xs = X[St].cpu().numpy()
    del X
    torch.cuda.empty_cache()
    idx_s = sk.indices[St].cpu().numpy().astype(np.uint32)
    val_s = sk.values[St].cpu().numpy()
    # the sampled rows' indices (global columns) and fp64 values against the oracle
    for t in range(0, len(S), 500):
        assert np.array_equal(idx_s[t], O.indices_block(plan.master_seed, int(S[t]), int(S[t]) + 1, p, m)[0])
    Y = O.precondition_rows(Xs.astype(np.float64), p, O.HADAMARD, spec.sign_seed)
    assert np.array_equal(val_s, np.take_along_axis(Y, idx_s.astype(np.int64), axis=1))
    del Y, Xs
    io_full = sk.host_indices()
    vo_full = sk.host_values()
    chosen = np.random.default_rng(SEED).choice(n, K, replace=False)
    ops = skc.SketchKMeans(sk)
    mu = ops.init_centers(chosen)
    mu0 = mu.clone()
    lab = [torch.empty(n, dtype=torch.int32, device=dev) for _ in range(2)]
    d2min = torch.empty(n, dtype=torch.float64, device=dev)
    out = torch.zeros(2, dtype=torch.int64, device=dev)
    d2max = torch.zeros(1, dtype=torch.float64, device=dev)
    prev, iters, updates = None, 0, 0
    for it in range(c["iters"]):
        cur = lab[it % 2]
        ops.assign(mu, prev, cur, d2min, out, d2max)
        mu_h = mu.cpu().numpy()
        lo, do = O.kmeans_assign(idx_s, val_s, mu_h, nthreads=NT)
        assert np.array_equal(cur[St].cpu().numpy(), lo), f"labels differ at iteration {it}"
        assert np.array_equal(d2min[St].cpu().numpy(), do), f"d2min differs at iteration {it}"
        iters += 1
        changed = int(out[0])
        if prev is not None and changed == 0:
            break
        prev = cur
        mu_next, counts, empty = ops.update(cur, mu)
        if it in (0, c["iters"] - 2):  # whole-job counts and centres against the oracle's update
            muo, co, eo = O.kmeans_update(io_full, vo_full, cur.cpu().numpy(), mu_h)
            assert np.array_equal(counts.cpu().numpy(), co), f"counts differ at iteration {it}"
            assert np.array_equal(mu_next.cpu().numpy(), muo), f"centres differ at iteration {it}"
            assert np.array_equal(empty.cpu().numpy().astype(bool), eo)
            updates += 1
        ops.reseed_at(mu_next, empty, out[1:2])
        mu = mu_next
    assert updates >= 1
    # the public loop follows the same trajectory
    labels, mu_l, traj, it_l, _ = ops.lloyd(mu0, c["iters"])
    assert it_l == iters and torch.equal(labels, cur)
    print(f"C5 Lloyd: {iters} iterations checked on 10^5 sampled points")
