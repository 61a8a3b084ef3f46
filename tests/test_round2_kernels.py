"""Round-2 kernels against the kernels they replace, bit for bit (both sides are pinned to the
reference elsewhere: K5 / K5s by the golden K-means trajectories, K3 by the golden covariances).

* K3 cov_flat_kernel (m <= 64, the default) vs the round-1 cov_band_kernel (SKC_COV_KERNEL=band):
  both sum the same fixed-point integers, so the triangles are bit-identical, including rows that
  take the exact fp64 path (values above tau) in every band, m = 2 (one pair per row) and m = 64
  (two full lane chunks).
* K5c (cooperative small-K assignment, tables in shared memory) vs K5s (one point per thread):
  labels, d2min, changed count and farthest point bit-identical for every lanes-per-point width
  H = ceil(K/2) = 1..8, ragged point counts and near-ties. Every shape keeps the padded tables and
  the row staging within K5c's shared-memory budget (16 p KC + 96 (32/H) m bytes <= 110 KB).
"""

import numpy as np
import pytest
import torch

from oracle import oracle as O

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def skc():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_1511_00152_b200 as skc

    return skc


def rel_fro(a, b):
    return float(np.linalg.norm(a - b) / np.linalg.norm(b))


@pytest.mark.parametrize("p,m,compute", [(256, 2, "f64"), (256, 33, "f32"), (1024, 51, "f64"), (1024, 64, "f32"),
                                         (512, 40, "f64")])
def test_flat_covariance_equals_band_kernel(skc, monkeypatch, p, m, compute):
    rng = np.random.default_rng(p * 100 + m)
    n = 7000
    X = (rng.standard_t(3, size=(p, n)) / np.sqrt(3.0)).astype(np.float32)
    X[:, 11] *= 1e3  # rows above tau: the exact fp64 path, in every band they reach
    X[:, 4000] *= 5e2
    spec = skc.PreconditionSpec.create("hadamard", p, 7)
    sk = skc.sketch_stream(X, spec, skc.SamplingPlan(8, p, m), compute=compute)
    monkeypatch.setenv("SKC_COV_PATH", "band")
    monkeypatch.setenv("SKC_COV_KERNEL", "band")
    Cb = skc.estimate_covariance(sk).matrix
    monkeypatch.setenv("SKC_COV_KERNEL", "flat")
    Cf = skc.estimate_covariance(sk).matrix
    assert np.array_equal(Cf, Cb)
    Co = O.estimate_covariance(sk.host_indices(), sk.host_values().astype(np.float64), p, nthreads=8)
    assert rel_fro(Cf, Co) < 1e-6


def _assign(skc, sk, mu, prev, coop, monkeypatch, reg=False):
    from paper_1511_00152_b200 import _lib

    L = _lib.lib()
    dev = mu.device
    n, m = sk.indices.shape
    K = mu.shape[1]
    vcode = _lib.F64 if sk.values.dtype == torch.float64 else _lib.F32
    ws = _lib.workspace(L.skc_kmeans_assign_workspace(n, sk.spec.p_pad, K), dev)
    labels = torch.empty(n, dtype=torch.int32, device=dev)
    d2min = torch.empty(n, dtype=torch.float64, device=dev)
    out = torch.zeros(2, dtype=torch.int64, device=dev)
    d2max = torch.zeros(1, dtype=torch.float64, device=dev)
    monkeypatch.setenv("SKC_ASSIGN_EXACT", "1")
    monkeypatch.setenv("SKC_ASSIGN_COOP", "1" if coop else "0")
    monkeypatch.setenv("SKC_ASSIGN_REG", "1" if reg else "0")
    _lib.call("skc_kmeans_assign", sk.indices.data_ptr(), sk.values.data_ptr(), vcode, n, m, mu.data_ptr(),
              sk.spec.p_pad, K, _lib.ptr(prev), labels.data_ptr(), d2min.data_ptr(), out.data_ptr(),
              d2max.data_ptr(), ws.data_ptr(), ws.numel(), _lib.stream_ptr(dev))
    torch.cuda.synchronize()
    return labels.cpu().numpy(), d2min.cpu().numpy(), out.cpu().numpy(), d2max.cpu().numpy()


@pytest.mark.parametrize("p,m,K,n,spread,compute", [
    (512, 26, 10, 20000, 2.0, "f64"),   # C2 shape (H = 5)
    (512, 26, 10, 3001, 0.02, "f64"),   # near-ties, ragged last warp step
    (256, 7, 1, 999, 1.0, "f64"),       # one centre (H = 1)
    (256, 1, 2, 1234, 1.0, "f32"),      # one kept coordinate, fp32 values
    (256, 64, 5, 4097, 1.0, "f64"),     # m = 64 (largest staged row), H = 3
    (512, 33, 7, 5000, 0.5, "f32"),     # H = 4
    (128, 12, 13, 777, 1.0, "f64"),     # H = 7
    (256, 40, 16, 6000, 1.0, "f64"),    # H = 8 (largest K of the small path)
    (256, 20, 11, 2500, 1.0, "f64"),    # H = 6
])
def test_k5c_equals_k5s(skc, monkeypatch, p, m, K, n, spread, compute):
    rng = np.random.default_rng(p + m + K + n)
    C = rng.standard_normal((p, K)) * spread
    lab = rng.integers(0, K, n)
    X = (C[:, lab] + rng.standard_normal((p, n))).astype(np.float32)
    spec = skc.PreconditionSpec.create("hadamard", p, 5)
    sk = skc.sketch_stream(X, spec, skc.SamplingPlan(6, spec.p_pad, m), compute=compute)
    dev = sk.indices.device
    mu = torch.as_tensor(rng.standard_normal((spec.p_pad, K)) * spread * 0.9, device=dev)
    prev = torch.as_tensor(rng.integers(0, K, n).astype(np.int32), device=dev)
    a = _assign(skc, sk, mu, prev, True, monkeypatch)
    b = _assign(skc, sk, mu, prev, False, monkeypatch)
    assert np.array_equal(a[0], b[0]), "labels"
    assert np.array_equal(a[1], b[1]), "d2min"
    assert np.array_equal(a[2], b[2]) and np.array_equal(a[3], b[3]), "changed / farthest point"


@pytest.mark.parametrize("p,m,K,n,spread,compute", [
    (512, 26, 10, 20000, 2.0, "f64"),   # C2 shape (H = 5, MT = 32)
    (512, 26, 10, 3001, 0.02, "f64"),   # near-ties, ragged last warp step
    (256, 7, 1, 999, 1.0, "f64"),       # one centre (H = 1, MT = 16)
    (256, 1, 2, 1234, 1.0, "f32"),      # one kept coordinate, fp32 values
    (256, 32, 5, 4097, 1.0, "f64"),     # m = 32 (largest register row), H = 3
    (512, 17, 7, 5000, 0.5, "f32"),     # H = 4, first m of MT = 32
    (128, 12, 13, 777, 1.0, "f64"),     # H = 7
    (256, 16, 16, 6000, 1.0, "f64"),    # H = 8 (largest K of the small path), m = MT = 16
    (256, 20, 11, 2500, 1.0, "f64"),    # H = 6
    (2048, 30, 9, 3000, 1.0, "f64"),    # a table above 100 KB (compact layout only)
    (256, 9, 14, 2222, 1.0, "f64"),     # H = 7: three components (4 + 2 + 1)
    (128, 5, 3, 1500, 1.0, "f32"),      # H = 2
    (256, 28, 8, 3333, 0.7, "f64"),     # H = 4, m = MT = 28
])
def test_k5r_equals_k5s(skc, monkeypatch, p, m, K, n, spread, compute):
    """K5r (mu in registers between the two halves of the chain, one table pass, products formed
    as (-2 v) mu) against K5s (the reference's term order with precomputed -2 mu and mu^2
    tables): labels, d2min, changed count and farthest point bit-identical, including centres and
    values with zeros, negative zeros and subnormal products."""
    rng = np.random.default_rng(p + m + K + n + 1)
    C = rng.standard_normal((p, K)) * spread
    lab = rng.integers(0, K, n)
    X = (C[:, lab] + rng.standard_normal((p, n))).astype(np.float32)
    X[:, ::7] = 0.0  # all-zero points: every product is a signed zero
    spec = skc.PreconditionSpec.create("hadamard", p, 5)
    sk = skc.sketch_stream(X, spec, skc.SamplingPlan(6, spec.p_pad, m), compute=compute)
    dev = sk.indices.device
    mu_h = rng.standard_normal((spec.p_pad, K)) * spread * 0.9
    mu_h[::5] = 0.0
    mu_h[1::5] = -0.0
    mu_h[2::11] *= 1e-160  # products and squares in the subnormal range
    mu = torch.as_tensor(mu_h, device=dev)
    prev = torch.as_tensor(rng.integers(0, K, n).astype(np.int32), device=dev)
    b = _assign(skc, sk, mu, prev, False, monkeypatch)
    for spread in ("1", "0"):  # the replicated conflict-free table (when it fits), and the compact one
        monkeypatch.setenv("SKC_ASSIGN_SPREAD", spread)
        a = _assign(skc, sk, mu, prev, False, monkeypatch, reg=True)
        assert np.array_equal(a[0], b[0]), "labels"
        assert np.array_equal(a[1], b[1]), "d2min"
        assert np.array_equal(a[2], b[2]) and np.array_equal(a[3], b[3]), "changed / farthest point"


@pytest.mark.parametrize("p,m,K,n,spread", [(512, 26, 10, 20000, 2.0), (256, 20, 12, 3000, 0.3), (2048, 40, 30, 4000, 1.0)])
def test_lloyd_fused_tail_equals_stepwise(skc, monkeypatch, p, m, K, n, spread):
    """The Lloyd graph's fused tail (objective + check in one block, the partial sums beside it on a
    second branch, centres + reseed + commit in one kernel with cluster sizes taken from the counts)
    against the kernel-per-step graph: labels, centres, trajectory and iteration count bit for bit,
    including iterations that reseed empty clusters (duplicate initial points)."""
    rng = np.random.default_rng(p + m + K)
    C = rng.standard_normal((p, K)) * spread
    X = (C[:, rng.integers(0, K, n)] + rng.standard_normal((p, n))).astype(np.float32)
    spec = skc.PreconditionSpec.create("hadamard", p, 3)
    sk = skc.sketch_stream(X, spec, skc.SamplingPlan(4, spec.p_pad, m))
    chosen = rng.choice(n, K, replace=False)
    chosen[1] = chosen[0]  # two equal centres: one of them empties and is reseeded
    chosen[K - 1] = chosen[0]
    res = {}
    for mode in ("0", "1"):
        monkeypatch.setenv("SKC_LLOYD_FUSED", mode)
        ops = skc.SketchKMeans(sk)
        labels, mu, traj, iters, _ = ops.lloyd(ops.init_centers(chosen), 12)
        res[mode] = (labels.cpu().numpy(), mu.cpu().numpy(), traj, iters)
    assert res["0"][3] == res["1"][3] and res["0"][2] == res["1"][2]
    assert np.array_equal(res["0"][0], res["1"][0])
    assert np.array_equal(res["0"][1], res["1"][1])
