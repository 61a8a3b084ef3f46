"""Covariance accumulation at extreme value scales (estimators.py:48-66 against the oracle).

The fixed-point paths (K3 banded, K3g global) scale each factor by 2^(S/2) with S taken from
the value statistics; K3t scales by the value maximum. Data far from unit scale, huge single
outliers and fp64 values outside the float range must still match the reference's fp64
covariance (the wide-range and huge-product cases take exact fp64 atomics).
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
    import paper_1511_00152_b200 as m

    return m


def rel_fro(a, b):
    s = np.abs(b).max()  # scale first: the Frobenius norm of 1e301 entries overflows fp64
    return float(np.linalg.norm((a - b) / s) / max(np.linalg.norm(b / s), 1e-300))


@pytest.mark.parametrize("path", ["b", "g", "t"])
@pytest.mark.parametrize("scale", [1e-20, 1e30])
@pytest.mark.parametrize("compute", ["f64", "f32"])
def test_extreme_data_scales(skc, monkeypatch, path, scale, compute):
    monkeypatch.setenv("SKC_COV_PATH", path)
    p, n, m = 256, 3000, 25
    X = (np.random.default_rng(1).standard_normal((n, p)) * scale).astype(np.float32)
    spec = skc.PreconditionSpec.create("hadamard", p, sign_seed=3)
    plan = skc.SamplingPlan(4, p, m)
    sk = skc.sketch_stream(skc.RowSource(torch.as_tensor(X).cuda()), spec, plan, compute=compute)
    C = skc.estimate_covariance(sk).matrix
    Co = O.estimate_covariance(sk.host_indices(), sk.host_values(), p)
    assert np.isfinite(C).all()
    assert rel_fro(C, Co) < (1e-5 if path == "t" else 1e-6)


@pytest.mark.parametrize("path", ["b", "g"])
@pytest.mark.parametrize("scale", [1e-120, 1e150])
def test_fp64_values_outside_float_range(skc, monkeypatch, path, scale):
    # a hand-built fp64 sketch (test_estimators.py:22-29 style) with values no float holds
    monkeypatch.setenv("SKC_COV_PATH", path)
    p, n, m = 256, 2000, 20
    rng = np.random.default_rng(2)
    idx = np.sort(np.argsort(rng.random((n, p)), axis=1)[:, :m], axis=1)
    val = rng.standard_normal((n, m)) * scale
    spec = skc.PreconditionSpec.create("hadamard", p, sign_seed=1)
    sk = skc.SparseSketch.from_host(spec, n, idx, val)
    C = skc.estimate_covariance(sk).matrix
    Co = O.estimate_covariance(idx.astype(np.uint32), val, p)
    assert rel_fro(C, Co) < 1e-12  # exact fp64 products, only the summation order differs


@pytest.mark.parametrize("path", ["b", "g"])
def test_huge_outlier(skc, monkeypatch, path):
    # one value 1e12 x the rms: its products exceed the int64 fixed-point range and take the
    # fp64 path. (The rms-derived quantum then grows with the outlier: the entries away from
    # it keep an absolute error of ~2^-S, far inside the relative-Frobenius contract.)
    monkeypatch.setenv("SKC_COV_PATH", path)
    p, n, m = 256, 2000, 20
    rng = np.random.default_rng(3)
    idx = np.sort(np.argsort(rng.random((n, p)), axis=1)[:, :m], axis=1)
    val = rng.standard_normal((n, m))
    val[17, 3] = 1e12
    val[900, 0] = -3e9
    spec = skc.PreconditionSpec.create("hadamard", p, sign_seed=1)
    sk = skc.SparseSketch.from_host(spec, n, idx, val)
    C = skc.estimate_covariance(sk).matrix
    Co = O.estimate_covariance(idx.astype(np.uint32), val, p)
    assert rel_fro(C, Co) < 1e-9
