"""GPU parity: the CUDA path (through the C ABI) against the reference's golden
fixtures and the pinned CPU oracle.

Tolerances:
  indices, counts, labels          bit-exact
  fp64 sketch values, transforms   bit-exact
  mean                             1e-12 relative (parallel fp64 sum order)
  covariance                       1e-6 relative Frobenius (int32x2 fixed-point accumulator,
                                   ~1e-7 typical; the north_star bound is 1e-5)
  fp32 fast path                   values 2e-6 relative, covariance 1e-5 relative Frobenius
                                   (the north_star bound)
"""

import numpy as np
import pytest
import torch

from datagen import digest, mixture, spiked
from oracle import oracle as O

pytestmark = pytest.mark.gpu

LAMS = [50.0, 40.0, 30.0, 20.0, 10.0]
SEED = 2026


@pytest.fixture(scope="module")
def skc():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_1511_00152_b200 as skc

    return skc


def rel_fro(a, b):
    return float(np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-300))


# ---------------------------------------------------------------- L0 / L1
def test_signs_and_indices_bit_exact(skc, golden):
    g = golden("hash")
    for s, p in [(1, 16), (77, 1024), (123, 64), (0, 4096)]:
        assert np.array_equal(skc.PreconditionSpec.create("hadamard", p, s).signs(), g[f"signs_{s}_{p}"])
    for k, (ms, p, m, i0, i1) in enumerate(g["idx_meta"]):
        plan = skc.SamplingPlan(master_seed=int(ms), p=int(p), m=int(m))
        assert np.array_equal(plan.indices_block(int(i0), int(i1)), g[f"idx_{k}"]), (ms, p, m, i0, i1)


def test_survey_known_answers(skc):
    plan = skc.SamplingPlan(2, 16, 4)
    assert plan.indices_block(0, 4).tolist() == [[3, 7, 11, 15], [0, 2, 11, 13], [4, 5, 7, 8], [3, 12, 13, 15]]
    assert skc.SamplingPlan(2, 256, 25).indices(0).tolist() == [
        25, 27, 30, 48, 52, 64, 85, 114, 118, 121, 128, 139, 140, 146, 168, 189, 200, 214, 218, 223, 231, 235, 238,
        249, 254]


def test_fwht_known_answers(skc, golden):
    g = golden("transform")
    assert np.array_equal(skc.fwht_inplace(np.array([1.0, 0.0])), g["fwht_2"])
    assert np.array_equal(skc.fwht_inplace(np.array([1.0, 1.0, 1.0, 1.0])), g["fwht_4"])
    H = np.column_stack([skc.fwht_inplace(np.eye(16)[:, j].copy()) for j in range(16)])
    assert np.array_equal(H, g["hadamard_16"])
    v = np.random.default_rng(0).standard_normal(8)
    assert np.abs(skc.fwht_inplace(skc.fwht_inplace(v.copy())) - v).max() < 1e-12
    with pytest.raises(skc.DimensionError):
        skc.fwht_inplace(np.ones(3))


def test_precondition_bit_exact(skc, golden):
    g = golden("transform")
    for k, (kind, p, p_pad, seed) in enumerate(g["pre_meta"]):
        spec = skc.PreconditionSpec.create("hadamard" if kind == 0 else "none", int(p), int(seed))
        X = g[f"pre_X_{k}"]
        assert np.array_equal(skc.precondition_columns(X, spec), g[f"pre_Y_{k}"]), (kind, p)
        assert np.array_equal(skc.unprecondition_columns(g[f"pre_Y_{k}"], spec), g[f"unpre_{k}"])
        # device in -> device out
        Yd = skc.precondition_columns(torch.as_tensor(X).cuda(), spec)
        assert Yd.is_cuda and np.array_equal(Yd.cpu().numpy(), g[f"pre_Y_{k}"])
        # vector path equals the batch path bit for bit (test_transform.py:137-144)
        assert np.array_equal(skc.precondition(X[:, 0], spec), g[f"pre_Y_{k}"][:, 0])


def test_spec_errors(skc):
    with pytest.raises(skc.ParameterError):
        skc.PreconditionSpec.create("fourier", 8)
    with pytest.raises(skc.DimensionError):
        skc.PreconditionSpec(kind="hadamard", sign_seed=0, p=5, p_pad=6)
    with pytest.raises(skc.DimensionError):
        skc.precondition(np.ones(11), skc.PreconditionSpec.create("hadamard", 10))
    with pytest.raises(skc.ParameterError):  # dct is outside the GPU hot path
        skc.precondition(np.ones(8), skc.PreconditionSpec.create("dct", 8))


# ---------------------------------------------------------------- L2 sketch
def _sketch_case(g, name):
    kind, p, p_pad, n, m, ss, ms, k = (int(v) for v in g[f"{name}_meta"])
    X = spiked(SEED + p + n, p, n, LAMS[: max(1, min(5, p - 1))])
    if name == "odd":
        X[:, 17] = 0.0
    assert digest(X) == str(g[f"{name}_X_sha"])
    return X, ("hadamard" if kind == 0 else "none"), p, p_pad, n, m, ss, ms, k


NAMES = ["c1", "c3", "c4", "odd", "none", "full", "tiny", "p32", "c5", "c2"]


@pytest.mark.parametrize("name", NAMES)
def test_sketch_f64_bit_exact_and_estimators(skc, golden, name):
    g = golden("sketch")
    X, kind, p, p_pad, n, m, ss, ms, k = _sketch_case(g, name)
    spec = skc.PreconditionSpec.create(kind, p, ss)
    plan = skc.SamplingPlan(ms, p_pad, m)
    sk = skc.sketch_stream(skc.ArraySource(X, chunk_cols=97), spec, plan, compute="f64")
    assert np.array_equal(sk.host_indices(), g[f"{name}_idx"])
    assert np.array_equal(sk.host_values(), g[f"{name}_val"])
    mean = skc.estimate_mean(sk)
    assert np.abs(mean - g[f"{name}_mean"]).max() <= 1e-12 * max(1.0, np.abs(g[f"{name}_mean"]).max())
    if m >= 2:
        C = skc.estimate_covariance(sk).matrix
        if f"{name}_cov" in g:
            assert rel_fro(C, g[f"{name}_cov"]) < 1e-6
        else:
            sel = g[f"{name}_cov_sel"]
            assert np.abs(C.diagonal() - g[f"{name}_cov_diag"]).max() < 1e-6 * np.abs(g[f"{name}_cov_diag"]).max()
            assert np.abs(C[sel[0], sel[1]] - g[f"{name}_cov_selval"]).max() < 1e-6 * float(g[f"{name}_cov_fro"])
            assert abs(np.linalg.norm(C) - float(g[f"{name}_cov_fro"])) < 1e-6 * float(g[f"{name}_cov_fro"])
        U = skc.principal_components(sk, k)
        ref = g[f"{name}_pcs"]
        sgn = np.sign(np.sum(U * ref, axis=0))  # eigenvector sign is parity-unpinned
        assert np.abs(U * sgn - ref).max() < 1e-6
        # device eigensolve (cuSOLVER): same eigenvectors up to sign, eigensolver rounding
        Ud = skc.principal_components(sk, k, solver="device")
        sgn = np.sign(np.sum(Ud * U, axis=0))
        assert np.abs(Ud * sgn - U).max() < 1e-7


@pytest.mark.parametrize("name", ["c1", "c3", "c4", "c5", "c2"])
def test_sketch_f32_fast_path(skc, golden, name):
    g = golden("sketch")
    X, kind, p, p_pad, n, m, ss, ms, k = _sketch_case(g, name)
    spec = skc.PreconditionSpec.create(kind, p, ss)
    plan = skc.SamplingPlan(ms, p_pad, m)
    sk = skc.sketch_stream(X, spec, plan, compute="f32")
    assert sk.values.dtype == torch.float32
    assert np.array_equal(sk.host_indices(), g[f"{name}_idx"])  # indices stay bit-exact
    ref = g[f"{name}_val"]
    scale = np.abs(ref).max()
    assert np.abs(sk.host_values() - ref).max() <= 2e-6 * scale
    C = skc.estimate_covariance(sk).matrix
    Co = O.estimate_covariance(g[f"{name}_idx"], ref, p_pad)
    assert rel_fro(C, Co) < 1e-5  # north_star tolerance


def test_chunk_invariance_and_column_equivalence(skc):
    # test_sketch.py:161-171, :182-190
    spec = skc.PreconditionSpec.create("hadamard", 50, sign_seed=2)
    plan = skc.plan_for(spec, 0.25, master_seed=6)
    X = np.random.default_rng(2).standard_normal((50, 1000))
    runs = [skc.sketch_stream(skc.ArraySource(X, chunk_cols=c), spec, plan) for c in (1, 7, 1000)]
    for sk in runs[1:]:
        assert torch.equal(sk.indices, runs[0].indices) and torch.equal(sk.values, runs[0].values)
    dev = skc.sketch_stream(torch.as_tensor(X).cuda(), spec, plan)
    assert torch.equal(dev.indices, runs[0].indices) and torch.equal(dev.values, runs[0].values)
    for i in (0, 11, 999):
        idx, val = skc.sketch_column(X[:, i], spec, plan, i)
        assert np.array_equal(idx, runs[0].host_indices()[i]) and np.array_equal(val, runs[0].host_values()[i])


def test_sharded_sketch_is_byte_identical(skc):
    spec = skc.PreconditionSpec.create("hadamard", 256, sign_seed=9)
    plan = skc.plan_for(spec, 25 / 256, master_seed=10)
    X = np.random.default_rng(3).standard_normal((256, 3000)).astype(np.float32)
    full = skc.sketch_stream(X, spec, plan, compute="f32")
    parts = [skc.sketch_stream(X[:, a:b], spec, plan, compute="f32", col0=a) for a, b in [(0, 1234), (1234, 3000)]]
    assert torch.equal(torch.cat([q.indices for q in parts]), full.indices)
    assert torch.equal(torch.cat([q.values for q in parts]), full.values)


def test_sketch_edge_cases(skc):
    spec = skc.PreconditionSpec.create("hadamard", 8, sign_seed=1)
    idx, val = skc.sketch_column(np.zeros(8), spec, skc.SamplingPlan(5, 8, 3), 2)
    assert idx.shape == (3,) and np.array_equal(val, np.zeros(3))  # zero vector keeps m slots
    plan = skc.SamplingPlan(master_seed=1, p=6, m=6)
    assert np.array_equal(plan.indices(3), np.arange(6))
    sp = skc.PreconditionSpec.create("none", 5)
    idx, val = skc.sketch_column(np.array([5.0, 4.0, 3.0, 2.0, 1.0]), sp, skc.SamplingPlan(3, 5, 5), 0)
    assert np.array_equal(val, [5.0, 4.0, 3.0, 2.0, 1.0])
    with pytest.raises(skc.ParameterError):
        skc.SamplingPlan(master_seed=0, p=4, m=0)
    sn = skc.PreconditionSpec.create("none", 10)
    pn = skc.plan_for(sn, 0.5, master_seed=1)
    with pytest.raises(skc.DimensionError):
        skc.sketch_stream(np.zeros((11, 5)), sn, pn)
    with pytest.raises(skc.DimensionError):
        skc.sketch_stream(np.zeros((10, 5)), sn, skc.SamplingPlan(master_seed=0, p=9, m=2))

    class FlakySource:  # test_sketch.py:203-215
        p, n, passes = 10, 8, 0

        def chunks(self):
            self.passes += 1
            yield np.zeros((10, 4))
            yield np.zeros((9, 4))

    with pytest.raises(skc.DimensionError, match="offset 4"):
        skc.sketch_stream(FlakySource(), sn, pn)
    src = skc.ArraySource(np.random.default_rng(3).standard_normal((10, 30)), chunk_cols=4)
    skc.sketch_stream(src, sn, pn)
    assert src.passes == 1


def test_sampler_fallback_and_large_m(skc):
    # m near p, tiny p, and m with the all-candidates select: compare with the oracle
    for ms, p, m in [(3, 64, 63), (3, 128, 100), (8, 32, 16), (4, 1024, 700), (5, 4096, 2000), (6, 2, 1)]:
        plan = skc.SamplingPlan(ms, p, m)
        got = plan.indices_block(1000, 1300)
        assert np.array_equal(got, O.indices_block(ms, 1000, 1300, p, m)), (p, m)


# ---------------------------------------------------------------- L3a estimators (hand instances)
def test_estimators_hand_instances(skc):
    X = np.random.default_rng(3).standard_normal((6, 9))
    spec = skc.PreconditionSpec.create("none", 6)
    sk = skc.sketch_stream(X, spec, skc.SamplingPlan(4, 6, 6))
    est = skc.estimate_covariance(sk)
    # exact at m=p (test_estimators.py:69-76); K3's fixed-point quantum bounds the error at
    # ~6e-8 * tau^2 per product ("K3"), so the bound here is 1e-7, not 1e-12
    assert np.abs(est.matrix - X @ X.T / 9).max() < 1e-7 and est.n_used == 9
    x = np.array([[1.0], [2.0], [3.0]])
    acc = np.zeros((3, 3))
    for s in [(0, 1), (0, 2), (1, 2)]:
        hs = skc.SparseSketch.from_host(skc.PreconditionSpec.create("none", 3), 1, np.array([s]), x[list(s), 0][None, :])
        acc += skc.estimate_covariance(hs).matrix
    assert np.abs(acc / 3 - x @ x.T).max() < 1e-7
    with pytest.raises(skc.ParameterError):
        skc.estimate_covariance(skc.sketch_stream(X[:5], skc.PreconditionSpec.create("none", 5),
                                                  skc.SamplingPlan(7, 5, 1)))
    empty = skc.SparseSketch.from_host(skc.PreconditionSpec.create("none", 3), 0, np.zeros((0, 2)), np.zeros((0, 2)))
    with pytest.raises(skc.ParameterError):
        skc.estimate_mean(empty)


def test_covariance_heavy_tails_and_determinism(skc):
    # Student-t(3) noise exercises the outlier queue of the fixed-point accumulator
    rng = np.random.default_rng(11)
    p, n = 1024, 20000
    X = (rng.standard_t(3, size=(p, n)) / np.sqrt(3.0)).astype(np.float32)
    X[:, 5] *= 1e4  # one huge sample
    spec = skc.PreconditionSpec.create("hadamard", p, 3)
    plan = skc.SamplingPlan(4, p, 51)
    sk = skc.sketch_stream(X, spec, plan, compute="f64")
    C1 = skc.estimate_covariance(sk).matrix
    C2 = skc.estimate_covariance(sk).matrix
    assert np.array_equal(C1, C2)  # deterministic
    Co = O.estimate_covariance(sk.host_indices(), sk.host_values(), p, nthreads=8)
    assert rel_fro(C1, Co) < 1e-6


@pytest.mark.parametrize("p,m", [(512, 26), (2048, 40)])
def test_covariance_paths_bit_identical(skc, monkeypatch, p, m):
    # banded shared-memory accumulation and the L2-resident global path sum the same
    # fixed-point integers: the results are bit-identical, including the outlier path
    rng = np.random.default_rng(p)
    n = 6000
    X = (rng.standard_t(3, size=(p, n)) / np.sqrt(3.0)).astype(np.float32)
    X[:, 7] *= 1e3
    spec = skc.PreconditionSpec.create("hadamard", p, 1)
    sk = skc.sketch_stream(X, spec, skc.SamplingPlan(2, p, m), compute="f32")
    monkeypatch.setenv("SKC_COV_PATH", "band")
    Cb = skc.estimate_covariance(sk).matrix
    monkeypatch.setenv("SKC_COV_PATH", "global")
    Cg = skc.estimate_covariance(sk).matrix
    assert np.array_equal(Cb, Cg)
    Co = O.estimate_covariance(sk.host_indices(), sk.host_values().astype(np.float64), p, nthreads=8)
    assert rel_fro(Cg, Co) < 1e-6


def test_covariance_split_launches(skc, monkeypatch):
    # inputs beyond 2^31 elements per row group run as several launches; force the split
    # on a small input (fixed-point sums per launch, fp64 sum of launches: 1e-12)
    rng = np.random.default_rng(12)
    p, n = 256, 9000
    X = rng.standard_normal((p, n)).astype(np.float32)
    spec = skc.PreconditionSpec.create("hadamard", p, 5)
    sk = skc.sketch_stream(X, spec, skc.SamplingPlan(6, p, 20), compute="f32")
    C1 = skc.estimate_covariance(sk).matrix
    monkeypatch.setenv("SKC_COV_SPLIT_ROWS", "2500")
    C2 = skc.estimate_covariance(sk).matrix
    assert rel_fro(C2, C1) < 1e-12
    Co = O.estimate_covariance(sk.host_indices(), sk.host_values().astype(np.float64), p, nthreads=8)
    assert rel_fro(C2, Co) < 1e-6


# ---------------------------------------------------------------- L3b K-means
@pytest.mark.parametrize("name", ["c2", "c5", "small", "empty"])
@pytest.mark.parametrize("compute", ["f64"])
def test_kmeans_trajectory_bit_exact(skc, golden, name, compute):
    g = golden("kmeans")
    p, p_pad, n, K, m, max_iter, ss, ms = (int(v) for v in g[f"{name}_meta"])
    X = mixture(SEED + p + K, p, n, K, 2.0 if name != "empty" else 0.3)
    spec = skc.PreconditionSpec.create("hadamard", p, ss)
    sk = skc.sketch_stream(X, spec, skc.SamplingPlan(ms, p_pad, m), compute=compute)
    assert digest(sk.host_indices()) == str(g[f"{name}_idx_sha"])
    assert digest(sk.host_values()) == str(g[f"{name}_val_sha"])
    ops = skc.SketchKMeans(sk)
    mu0 = ops.init_centers(g[f"{name}_chosen"])
    labels, mu, traj, iters, _ = ops.lloyd(mu0, max_iter)
    assert iters == g[f"{name}_labels"].shape[0]
    assert np.array_equal(labels.cpu().numpy(), g[f"{name}_labels"][-1])  # bit-exact labels
    assert traj == g[f"{name}_traj"].tolist()  # bit-exact objective trajectory
    assert np.abs(mu.cpu().numpy() - g[f"{name}_mu_final"]).max() <= 1e-12 * np.abs(g[f"{name}_mu_final"]).max()
    res = skc.sparsified_kmeans(X, K, m / p_pad, max_iter=max_iter, init=g[f"{name}_chosen"], seed=0)
    assert res.diagnostics["passes"] == 1


def test_kmeans_each_iteration_against_oracle(skc, golden):
    g = golden("kmeans")
    p, p_pad, n, K, m, max_iter, ss, ms = (int(v) for v in g["small_meta"])
    X = mixture(SEED + p + K, p, n, K, 2.0)
    spec = skc.PreconditionSpec.create("hadamard", p, ss)
    sk = skc.sketch_stream(X, spec, skc.SamplingPlan(ms, p_pad, m))
    idx, val = sk.host_indices(), sk.host_values()
    ops = skc.SketchKMeans(sk)
    mu = ops.init_centers(g["small_chosen"])
    lab = torch.empty(n, dtype=torch.int32, device="cuda")
    d2 = torch.empty(n, dtype=torch.float64, device="cuda")
    out = torch.zeros(2, dtype=torch.int64, device="cuda")
    mx = torch.zeros(1, dtype=torch.float64, device="cuda")
    for it in range(g["small_labels"].shape[0] - 1):
        ops.assign(mu, None, lab, d2, out, mx)
        lo, do = O.kmeans_assign(idx, val, mu.cpu().numpy())
        assert np.array_equal(lab.cpu().numpy(), lo) and np.array_equal(d2.cpu().numpy(), do)
        assert int(out[1]) == int(np.argmax(do)) and float(mx) == do.max()
        mu_next, counts, empty = ops.update(lab, mu)
        mo, co, eo = O.kmeans_update(idx, val, lo, mu.cpu().numpy())
        assert np.array_equal(counts.cpu().numpy(), co) and np.array_equal(empty.cpu().numpy().astype(bool), eo)
        assert np.abs(mu_next.cpu().numpy() - mo).max() <= 1e-13 * max(1.0, np.abs(mo).max())
        mu = torch.as_tensor(mo, device="cuda")  # continue from the oracle's centres


def test_kmeans_hand_instances(skc):
    A = skc.Assignments
    sn = lambda p: skc.PreconditionSpec.create("none", p)  # noqa: E731
    sk = skc.SparseSketch.from_host(sn(4), 1, np.array([[0, 2]]), np.array([[1.0, 2.0]]))
    cs = skc.CenterSet(K=2, centers=np.array([[1.0, 0.0], [9.0, 9.0], [2.5, 2.0], [9.0, 9.0]]), domain="preconditioned")
    assert skc.sparsified_assign(sk, 0, cs) == 0
    sk = skc.SparseSketch.from_host(sn(2), 1, np.array([[0, 1]]), np.array([[0.0, 0.0]]))
    assert skc.sparsified_assign(sk, 0, skc.CenterSet(K=3, centers=np.ones((2, 3)))) == 0  # tie -> lowest
    sk = skc.SparseSketch.from_host(sn(4), 3, np.array([[0, 1], [0, 2], [1, 3]]),
                                    np.array([[1.0, 2.0], [3.0, 4.0], [6.0, 8.0]]))
    c, cnt = skc.sparsified_update_centers(sk, A(labels=np.zeros(3, int)), K=1)
    assert np.array_equal(c.centers[:, 0], [2.0, 4.0, 4.0, 8.0]) and np.array_equal(cnt.counts[:, 0], [2, 2, 1, 1])
    sk = skc.SparseSketch.from_host(sn(3), 1, np.array([[0, 1]]), np.array([[5.0, 6.0]]))
    c, _ = skc.sparsified_update_centers(sk, A(labels=np.array([0])), K=1,
                                         prev_centers=skc.CenterSet(K=1, centers=np.full((3, 1), 9.0)))
    assert np.array_equal(c.centers[:, 0], [5.0, 6.0, 9.0])
    sk = skc.SparseSketch.from_host(sn(2), 2, np.array([[0, 1], [0, 1]]), np.array([[1.0, 1.0], [3.0, 3.0]]))
    c, cnt = skc.sparsified_update_centers(sk, A(labels=np.array([0, 0])), K=2,
                                           prev_centers=skc.CenterSet(K=2, centers=np.array([[4.0, 7.0], [4.0, 7.0]])))
    assert np.array_equal(c.centers[:, 1], [7.0, 7.0]) and cnt.counts[:, 1].sum() == 0


def test_kmeanspp_matches_oracle_choice(skc):
    X = mixture(77, 32, 400, 4, 3.0)
    spec = skc.PreconditionSpec.create("hadamard", 32, 1)
    sk = skc.sketch_stream(X, spec, skc.SamplingPlan(2, 32, 12))
    from paper_1511_00152_b200.kmeanspp import kmeanspp_select, restart_rng, pp_select

    ops = skc.SketchKMeans(sk)
    idx, val = sk.host_indices(), sk.host_values()
    colsq = np.array([O.pairwise_sum(v * v) for v in val])

    def d2_host(c):
        W = np.zeros((400, 32))
        W[np.arange(400)[:, None], idx.astype(int)] = val
        cross = np.array([sum(val[i, t] * W[c, idx[i, t]] for t in range(12)) for i in range(400)])
        return (32 / 12) * np.clip(colsq + colsq[c] - 2.0 * cross, 0.0, None)

    for r in range(3):
        assert kmeanspp_select(ops, 4, 5, r) == pp_select(400, 4, restart_rng(5, r), d2_host)
    res = skc.sparsified_kmeans(X, 4, 12 / 32, n_init=2, seed=5)
    curve = res.diagnostics["objective_curve"]
    assert all(b <= a * (1 + 1e-9) for a, b in zip(curve, curve[1:]))


def test_stream_moments_matches_one_shot(skc):
    # streamed estimators (no stored sketch, copies overlapped) agree with the one-shot
    # sketch: same mean accumulator order per chunk (1e-12), covariance per-chunk fixed point
    rng = np.random.default_rng(21)
    p, n = 512, 30000
    X = rng.standard_normal((p, n)).astype(np.float32)
    spec = skc.PreconditionSpec.create("hadamard", p, 8)
    plan = skc.SamplingPlan(9, p, 26)
    sk = skc.sketch_stream(X, spec, plan, compute="f32")
    C1 = skc.estimate_covariance(sk).matrix
    host = torch.from_numpy(np.ascontiguousarray(X.T)).pin_memory()
    for src in (skc.RowSource(host, chunk_cols=7000), skc.ArraySource(X, chunk_cols=4096)):
        mom = skc.stream_moments(src, spec, plan, compute="f32")
        assert mom.n == n
        C2 = skc.covariance_from_moments(mom, p, plan.m, n).cpu().numpy()
        assert rel_fro(C2, C1) < 1e-7
        mean = skc.mean_from_moments(mom, spec, plan.m, n).cpu().numpy()
        assert np.abs(mean - skc.estimate_mean(sk)).max() < 1e-12 * max(1.0, np.abs(mean).max())


@pytest.mark.parametrize("sampler,kind", [("oracle", "hadamard"), ("philox", "hadamard"), ("oracle", "none")])
def test_stream_moments_native_equals_python_loop(skc, sampler, kind):
    # pinned host rows take the C++ chunk loop (skc_stream_moments); a pageable source the
    # Python loop: same kernels, same chunking, bit-identical partial sums
    rng = np.random.default_rng(31)
    p, n = 300, 20000
    X = rng.standard_normal((n, p)).astype(np.float32)
    spec = skc.PreconditionSpec.create(kind, p, 4)
    plan = skc.SamplingPlan(6, spec.p_pad, 20, sampler=sampler)
    pinned = torch.from_numpy(X).pin_memory()
    a = skc.stream_moments(skc.RowSource(pinned, chunk_cols=3000), spec, plan, compute="f32")
    b = skc.stream_moments(skc.RowSource(torch.from_numpy(X), chunk_cols=3000), spec, plan, compute="f32")
    assert a.n == b.n == n
    assert torch.equal(a.acc, b.acc) and torch.equal(a.stats, b.stats) and torch.equal(a.tri, b.tri)


@pytest.mark.parametrize("n", [1, 7, 8, 127, 128, 129, 1000, 4097, 200000, 3000001, 10000000])
def test_pairwise_sum_bit_exact(skc, n):
    """skc_pairwise_sum reproduces numpy's pairwise float64 sum (ndarray.sum) bit for bit."""
    from paper_1511_00152_b200 import _lib

    L = _lib.lib()
    x = np.random.default_rng(n).standard_normal(n) * 10.0 ** np.random.default_rng(n + 1).integers(-3, 4, n)
    xd = torch.as_tensor(x, device="cuda")
    out = torch.zeros(1, dtype=torch.float64, device="cuda")
    ws = _lib.workspace(L.skc_pairwise_sum_workspace(n), xd.device)
    _lib.call("skc_pairwise_sum", xd.data_ptr(), n, out.data_ptr(), ws.data_ptr(), ws.numel(), _lib.stream_ptr(xd.device))
    assert float(out.item()) == float(x.sum())


def test_sparsified_assign_near_ties_match_reference_formula(skc):
    # cluster.py:306-311 evaluates ((val[:, None] - mu[idx]) ** 2).sum(axis=0); with tight centres
    # and |v| ~ 1e3 the CSR x dense order of the Lloyd assignment would break near-ties
    # differently, so the single-column op must use the reference's own order
    rng = np.random.default_rng(5)
    p, n, m, K = 64, 400, 16, 12
    idx = np.sort(np.argsort(rng.random((n, p)), axis=1)[:, :m], axis=1)
    val = 1e3 + rng.standard_normal((n, m)) * 1e-3
    mu = 1e3 + rng.standard_normal((p, K)) * 1e-3
    spec = skc.PreconditionSpec.create("hadamard", p, sign_seed=1)
    sk = skc.SparseSketch.from_host(spec, n, idx, val)
    cs = skc.CenterSet(K=K, centers=mu, domain="preconditioned")
    for i in range(0, n, 7):
        diff = val[i][:, None] - mu[idx[i], :]
        want = int(np.argmin((diff * diff).sum(axis=0)))
        assert skc.sparsified_assign(sk, i, cs) == want
