"""Two-pass sparsified K-means (cluster.py:407-456) on the GPU.

Against the reference's own results (tests/golden/make_golden.py twopass): the first pass
matches bit for bit (same sketch, K-means++ draws and Lloyd arithmetic). Second-pass
labels must match exactly (well-separated, no near-ties). Means and the objective agree
to 1e-12 relative, since BLAS and our kernels sum in different orders.
"""

import numpy as np
import pytest
import torch

from datagen import digest, mixture

pytestmark = pytest.mark.gpu
SEED = 2026


@pytest.fixture(scope="module")
def skc():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_1511_00152_b200 as skc

    return skc


def _case(golden, name):
    g = golden("twopass")
    p, n, K, n_init, seed, chunk, max_iter = (int(v) for v in g[f"{name}_cfg"])
    scale, gamma = (float(v) for v in g[f"{name}_f"])
    X = mixture(SEED + 17 * p + K, p, n, K, scale).astype(np.float64)
    assert digest(X) == str(g[f"{name}_X_sha"])
    return g, X, p, n, K, n_init, seed, chunk, max_iter, gamma, str(g[f"{name}_kind"])


@pytest.mark.parametrize("name", ["sep", "mid", "none", "big"])
def test_two_pass_matches_reference(skc, golden, name):
    g, X, p, n, K, n_init, seed, chunk, max_iter, gamma, kind = _case(golden, name)
    src = skc.ArraySource(X, chunk_cols=chunk)
    res = skc.sparsified_kmeans_two_pass(src, K, gamma, max_iter=max_iter, n_init=n_init, seed=seed, kind=kind,
                                         chunk_cols=chunk)
    assert src.passes == 2 and res.diagnostics["passes"] == 2
    assert res.diagnostics["first_pass_objective"] == pytest.approx(float(g[f"{name}_first_objective"]), rel=1e-12)
    assert np.array_equal(res.assignments.labels, g[f"{name}_labels"])
    ref_c = g[f"{name}_centers"]
    assert np.abs(res.centers.centers - ref_c).max() <= 1e-12 * max(1.0, np.abs(ref_c).max())
    assert res.objective == pytest.approx(float(g[f"{name}_objective"]), rel=1e-12)


def test_two_pass_semantics_exact(skc):
    # pass 2 averages the first-pass clusters and re-assigns against the first-pass
    # centres, nothing more (the reference's test_two_pass_semantics_exact)
    X = mixture(SEED + 5, 12, 200, 3, 3.0).astype(np.float64)
    first = skc.sparsified_kmeans(X, 3, gamma=0.4, n_init=2, seed=21)
    second = skc.sparsified_kmeans_two_pass(X, 3, gamma=0.4, n_init=2, seed=21)
    lab1 = first.assignments.labels
    mu_hat = first.centers.centers
    for k in range(3):
        assert np.allclose(second.centers.centers[:, k], X[:, lab1 == k].mean(axis=1), rtol=0, atol=1e-12)
    d2 = ((X[:, :, None] - mu_hat[:, None, :]) ** 2).sum(axis=0)
    assert np.array_equal(second.assignments.labels, np.argmin(d2, axis=1))
    assert second.objective == pytest.approx(float(d2.min(axis=1).sum()), rel=1e-10)


def test_two_pass_from_dense_file_fp32_rows(skc, tmp_path):
    # out-of-core source (DNSE1 f64) and device fp32 rows give the same second pass
    from paper_1511_00152_b200 import io as skio

    X = mixture(SEED + 9, 96, 3000, 6, 2.0).astype(np.float64)
    path = tmp_path / "x.dnse"
    skio.write_dense(path, X)
    a = skc.sparsified_kmeans_two_pass(skio.DenseFileSource(path, chunk_cols=700), 6, 0.25, n_init=2, seed=4,
                                       chunk_cols=700)
    b = skc.sparsified_kmeans_two_pass(X, 6, 0.25, n_init=2, seed=4, chunk_cols=700)
    assert np.array_equal(a.assignments.labels, b.assignments.labels)
    assert np.array_equal(a.centers.centers, b.centers.centers)
    assert a.objective == b.objective
    rows32 = torch.as_tensor(X.T.astype(np.float32), device="cuda")
    c = skc.sparsified_kmeans_two_pass(skc.RowSource(rows32), 6, 0.25, n_init=2, seed=4, compute="f32")
    assert (c.assignments.labels == b.assignments.labels).mean() > 0.99


@pytest.mark.parametrize("K,p,n,dt", [(100, 130, 4000, np.float32), (70, 64, 3000, np.float64), (17, 200, 2500, np.float32)])
def test_dense_kernels_many_centres(skc, K, p, n, dt):
    # K > 16 runs several 16-centre passes in K8, K > 64 several 64-cluster passes in K9;
    # checked against numpy in fp64: labels exact (separated points), sums to 1e-12
    from paper_1511_00152_b200 import _lib

    rng = np.random.default_rng(K + p)
    C = rng.standard_normal((K, p)) * 6.0
    lab_true = rng.integers(0, K, n)
    X = (C[lab_true] + rng.standard_normal((n, p))).astype(dt)
    mu = C + 0.01 * rng.standard_normal((K, p))
    dev = torch.device("cuda")
    Xd = torch.as_tensor(X, device=dev)
    mud = torch.as_tensor(mu, device=dev)
    L = _lib.lib()
    ws = _lib.workspace(L.skc_dense_assign_workspace(p, K), dev)
    labels = torch.empty(n, dtype=torch.int32, device=dev)
    d2 = torch.empty(n, dtype=torch.float64, device=dev)
    st = _lib.stream_ptr(dev)
    _lib.call("skc_dense_assign", Xd.data_ptr(), _lib.dtype_code(Xd), p, n, p, mud.data_ptr(), K, ws.data_ptr(),
              labels.data_ptr(), d2.data_ptr(), st)
    Xf = X.astype(np.float64)
    D = (Xf * Xf).sum(1)[:, None] - 2.0 * Xf @ mu.T + (mu * mu).sum(1)[None, :]
    assert np.array_equal(labels.cpu().numpy(), np.argmin(D, axis=1))
    assert np.allclose(d2.cpu().numpy(), np.clip(D.min(axis=1), 0, None), rtol=1e-10, atol=1e-8)
    lab = torch.as_tensor(lab_true.astype(np.int32), device=dev)
    sums = torch.zeros((K, p), dtype=torch.float64, device=dev)
    counts = torch.zeros(K, dtype=torch.int64, device=dev)
    ws2 = _lib.workspace(L.skc_dense_sums_workspace(n, p, K), dev)
    _lib.call("skc_dense_sums", Xd.data_ptr(), _lib.dtype_code(Xd), p, n, p, lab.data_ptr(), K, sums.data_ptr(),
              counts.data_ptr(), ws2.data_ptr(), st)
    ref = np.zeros((K, p))
    np.add.at(ref, lab_true, Xf)
    assert np.array_equal(counts.cpu().numpy(), np.bincount(lab_true, minlength=K))
    assert np.abs(sums.cpu().numpy() - ref).max() <= 1e-12 * max(1.0, np.abs(ref).max())
