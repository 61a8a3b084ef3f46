"""K5f (fp32 filter) and K5t (tensor-core bf16 filter, kmeans_tc.cu), each followed by fp64
verification, against the exact assignment K5.

K5f runs when the packed (p, K) table does not fit shared memory (C5: p=2048, K=100). Its
labels, d2min, changed count and farthest point must equal K5's bit for bit (K5 is pinned
to the reference by the trajectory tests), including near-ties: clusters whose centres sit
close together make many points' distances to two centres agree to within the fp32 error
bound, so the verify step decides them.
"""

import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def skc():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_1511_00152_b200 as skc

    return skc


def _assign(skc, sk, mu, prev, exact, monkeypatch):
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
    monkeypatch.setenv("SKC_ASSIGN_EXACT", "1" if exact else "0")
    _lib.call("skc_kmeans_assign", sk.indices.data_ptr(), sk.values.data_ptr(), vcode, n, m, mu.data_ptr(),
              sk.spec.p_pad, K, _lib.ptr(prev), labels.data_ptr(), d2min.data_ptr(), out.data_ptr(),
              d2max.data_ptr(), ws.data_ptr(), ws.numel(), _lib.stream_ptr(dev))
    torch.cuda.synchronize()
    return labels.cpu().numpy(), d2min.cpu().numpy(), out.cpu().numpy(), d2max.cpu().numpy()


@pytest.mark.parametrize("p,m,K,n,spread,compute", [
    (2048, 102, 100, 20000, 3.0, "f64"),   # C5 shape
    (2048, 102, 100, 20000, 0.05, "f64"),  # centres nearly on top of each other: near-ties
    (1024, 51, 33, 9000, 1.0, "f32"),      # fp32 sketch values, ragged K
    (512, 200, 256, 4000, 2.0, "f64"),     # largest K, m > 128 (pairwise colsq on one lane)
])
def test_filter_equals_exact(skc, monkeypatch, p, m, K, n, spread, compute):
    rng = np.random.default_rng(p + K)
    C = rng.standard_normal((p, K)) * spread
    lab = rng.integers(0, K, n)
    X = (C[:, lab] + rng.standard_normal((p, n))).astype(np.float32)
    spec = skc.PreconditionSpec.create("hadamard", p, 3)
    sk = skc.sketch_stream(X, spec, skc.SamplingPlan(4, spec.p_pad, m), compute=compute)
    dev = sk.indices.device
    mu = torch.as_tensor(rng.standard_normal((spec.p_pad, K)) * spread * 0.9, device=dev)
    prev = torch.as_tensor(rng.integers(0, K, n).astype(np.int32), device=dev)
    a = _assign(skc, sk, mu, prev, True, monkeypatch)
    b = _assign(skc, sk, mu, prev, False, monkeypatch)
    assert np.array_equal(a[0], b[0]), "labels"
    assert np.array_equal(a[1], b[1]), "d2min"
    assert np.array_equal(a[2], b[2]) and np.array_equal(a[3], b[3]), "changed / farthest point"


def _assign_tc(skc, sk, mu, prev):
    from paper_1511_00152_b200 import _lib

    L = _lib.lib()
    dev = mu.device
    n, m = sk.indices.shape
    K, p_pad = mu.shape[1], sk.spec.p_pad
    assert L.skc_kmeans_tc_supported(p_pad, K, m) == 1
    vcode = _lib.F64 if sk.values.dtype == torch.float64 else _lib.F32
    prep = _lib.workspace(L.skc_kmeans_tc_prepare_workspace(n, m, p_pad), dev)
    st = _lib.stream_ptr(dev)
    _lib.call("skc_kmeans_tc_prepare", sk.indices.data_ptr(), sk.values.data_ptr(), vcode, n, m, p_pad,
              prep.data_ptr(), prep.numel(), st)
    ws = _lib.workspace(L.skc_kmeans_assign_tc_workspace(n, p_pad, K), dev)
    labels = torch.empty(n, dtype=torch.int32, device=dev)
    d2min = torch.empty(n, dtype=torch.float64, device=dev)
    out = torch.zeros(2, dtype=torch.int64, device=dev)
    d2max = torch.zeros(1, dtype=torch.float64, device=dev)
    _lib.call("skc_kmeans_assign_tc", sk.indices.data_ptr(), sk.values.data_ptr(), vcode, n, m, mu.data_ptr(), p_pad,
              K, _lib.ptr(prev), labels.data_ptr(), d2min.data_ptr(), out.data_ptr(), d2max.data_ptr(),
              prep.data_ptr(), ws.data_ptr(), ws.numel(), st)
    torch.cuda.synchronize()
    return labels.cpu().numpy(), d2min.cpu().numpy(), out.cpu().numpy(), d2max.cpu().numpy()


@pytest.mark.parametrize("p,m,K,n,spread,compute,init", [
    (2048, 102, 100, 20000, 3.0, "f64", "dense"),   # C5 shape
    (2048, 102, 100, 20000, 3.0, "f64", "points"),  # sparse initial centres: most points unresolved
    (2048, 102, 100, 9001, 0.05, "f64", "dense"),   # near-ties, ragged tile pairs
    (1024, 51, 33, 9000, 1.0, "f32", "dense"),      # fp32 sketch values, ragged K
    (512, 200, 128, 4000, 2.0, "f64", "dense"),     # largest K, m > 128
    (256, 25, 1, 700, 1.0, "f64", "dense"),         # one centre
    (4096, 82, 64, 3000, 2.0, "f32", "dense"),      # C4 shape (128 chunks per tile pair)
    (512, 1, 17, 2000, 1.0, "f64", "dense"),        # one kept coordinate per point
])
def test_tc_filter_equals_exact(skc, monkeypatch, p, m, K, n, spread, compute, init):
    rng = np.random.default_rng(p + K + n)
    C = rng.standard_normal((p, K)) * spread
    lab = rng.integers(0, K, n)
    X = (C[:, lab] + rng.standard_normal((p, n))).astype(np.float32)
    spec = skc.PreconditionSpec.create("hadamard", p, 3)
    sk = skc.sketch_stream(X, spec, skc.SamplingPlan(4, spec.p_pad, m), compute=compute)
    dev = sk.indices.device
    if init == "points":
        mu = skc.SketchKMeans(sk).init_centers(rng.choice(n, K, replace=False))
    else:
        mu = torch.as_tensor(rng.standard_normal((spec.p_pad, K)) * spread * 0.9, device=dev)
    prev = torch.as_tensor(rng.integers(0, K, n).astype(np.int32), device=dev)
    a = _assign(skc, sk, mu, prev, True, monkeypatch)
    b = _assign_tc(skc, sk, mu, prev)
    assert np.array_equal(a[0], b[0]), "labels"
    assert np.array_equal(a[1], b[1]), "d2min"
    assert np.array_equal(a[2], b[2]) and np.array_equal(a[3], b[3]), "changed / farthest point"


@pytest.mark.parametrize("p,m,K,n", [(2048, 102, 100, 30000), (1024, 51, 7, 20001), (512, 26, 10, 90000),
                                     (256, 25, 256, 50000), (256, 30, 32, 40000), (128, 3, 1, 5000),
                                     (256, 25, 2, 70001), (256, 25, 20, 30000), (128, 16, 13, 33333),
                                     (128, 9, 5, 100000)])
def test_partials_paths_agree(skc, monkeypatch, p, m, K, n):
    """K6's exact paths (tiled counting sort, warp-per-coordinate walk, segmented label sort) agree bit for bit."""
    rng = np.random.default_rng(p * 7 + K)
    X = (rng.standard_normal((p, K))[:, rng.integers(0, K, n)] * 2 + rng.standard_normal((p, n))).astype(np.float32)
    spec = skc.PreconditionSpec.create("hadamard", p, 5)
    sk = skc.sketch_stream(X, spec, skc.SamplingPlan(6, spec.p_pad, m))
    ops = skc.SketchKMeans(sk)
    labels = torch.as_tensor(rng.integers(0, K, n).astype(np.int32), device=sk.indices.device)
    res = {}
    for path in ("seg", "walk", "tile"):
        monkeypatch.setenv("SKC_PARTIALS", path)
        ops._ws.pop(("seg", K), None)
        res[path] = [t.cpu().numpy() for t in ops.partials(labels, K)]
    for other in ("walk", "tile"):
        for a, b in zip(res["seg"], res[other]):
            assert np.array_equal(a, b), other


@pytest.mark.parametrize("scale", [1e-30, 1e-12, 1.0, 1e25])
def test_filters_at_extreme_scales(skc, monkeypatch, scale):
    """Both filters stay exact when the data sit far from unit scale (the fp32 / bf16 bounds hold
    only for colsq in [2^-90, 2^100]; outside it every centre is verified) and for all-zero points."""
    p, m, K, n = 1024, 51, 40, 6000
    rng = np.random.default_rng(11)
    C = rng.standard_normal((p, K)) * 3.0
    X = (C[:, rng.integers(0, K, n)] + rng.standard_normal((p, n))) * scale
    X[:, ::97] = 0.0  # some all-zero points (colsq = 0)
    X = X.astype(np.float32)
    spec = skc.PreconditionSpec.create("hadamard", p, 3)
    sk = skc.sketch_stream(X, spec, skc.SamplingPlan(4, spec.p_pad, m), compute="f64")
    dev = sk.indices.device
    mu = torch.as_tensor(rng.standard_normal((spec.p_pad, K)) * 2.7 * scale, device=dev)
    prev = torch.as_tensor(rng.integers(0, K, n).astype(np.int32), device=dev)
    a = _assign(skc, sk, mu, prev, True, monkeypatch)
    for b in (_assign(skc, sk, mu, prev, False, monkeypatch), _assign_tc(skc, sk, mu, prev)):
        assert np.array_equal(a[0], b[0]), "labels"
        assert np.array_equal(a[1], b[1]), "d2min"
        assert np.array_equal(a[2], b[2]) and np.array_equal(a[3], b[3]), "changed / farthest point"


@pytest.mark.parametrize("p,m,K,n,compute,init", [
    (2048, 102, 100, 20000, "f64", "points"),  # C5 shape: the first iteration from seeded points
    (1024, 51, 33, 9001, "f32", "points"),     # fp32 values, ragged K and n
    (512, 26, 256, 4000, "f64", "points"),     # the largest K of K5f
    (2048, 102, 100, 5000, "f64", "dense"),    # dense centres
])
def test_first_iteration_filter_equals_exact(skc, monkeypatch, p, m, K, n, compute, init):
    """The first Lloyd assignment (no previous labels) from seeded points, whose centres are
    sketch columns (nearly every point has near-ties): K5f's outputs equal K5's bit for bit."""
    rng = np.random.default_rng(p + 3 * K + n)
    C = rng.standard_normal((p, K)) * 3.0
    lab = rng.integers(0, K, n)
    X = (C[:, lab] + rng.standard_normal((p, n))).astype(np.float32)
    spec = skc.PreconditionSpec.create("hadamard", p, 3)
    sk = skc.sketch_stream(X, spec, skc.SamplingPlan(4, spec.p_pad, m), compute=compute)
    dev = sk.indices.device
    if init == "points":
        mu = skc.SketchKMeans(sk).init_centers(rng.choice(n, K, replace=False))
    else:
        mu = torch.as_tensor(rng.standard_normal((spec.p_pad, K)), device=dev)
    a = _assign(skc, sk, mu, None, True, monkeypatch)
    b = _assign(skc, sk, mu, None, False, monkeypatch)
    assert np.array_equal(a[0], b[0]), "labels"
    assert np.array_equal(a[1], b[1]), "d2min"
    assert np.array_equal(a[2], b[2]) and np.array_equal(a[3], b[3]), "changed / farthest point"
