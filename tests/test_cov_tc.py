"""K3t, the tensor-core covariance path (cov_tc.cu; north_star: "a tcgen05/TMEM GEMM over
zero-filled tiles when m/p is large").

Against the oracle's fp64 estimate_covariance (estimators.py:53-66) on the same sketch, at the
contract's 1e-5 relative Frobenius: products carry ~22 bits (fp16 hi/lo split) and are exact
in fp32, but the tensor core's fp32 accumulation truncates. Over one 1024-row window in
TMEM (192 accumulations) that biases sums by about -2e-8 per accumulation, -4e-6 at most
(measured, tools/covtc_probe.py); the windows then add in fp64. Shapes cover ragged
chunks, tiny n, every unit kind (diagonal and off-diagonal strips), heavy outliers, m/p up to
1/2 (where the banded path cannot run) and fp32/fp64 sketch values.
"""

import numpy as np
import pytest
import torch

from oracle import oracle as O

pytestmark = pytest.mark.gpu


def rel_fro(a, b):
    return float(np.linalg.norm(a - b) / np.linalg.norm(b))


@pytest.fixture(scope="module")
def skc():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_1511_00152_b200 as skc

    return skc


def _sketch(skc, p, m, n, seed, compute="f32", outlier=False):
    rng = np.random.default_rng(seed)
    X = (rng.standard_t(3, size=(p, n)) / np.sqrt(3.0)).astype(np.float32)
    if outlier:
        X[:, 7] *= 1e3
    spec = skc.PreconditionSpec.create("hadamard", p, seed + 1)
    return skc.sketch_stream(X, spec, skc.SamplingPlan(seed + 2, p, m), compute=compute)


def _oracle(sk, p):
    return O.estimate_covariance(sk.host_indices(), sk.host_values().astype(np.float64), p, nthreads=8)


@pytest.mark.parametrize(
    "p,m,n,compute,outlier",
    [
        (256, 64, 5000, "f32", False),
        (256, 128, 777, "f64", False),  # ragged last chunk
        (512, 64, 20000, "f32", True),  # heavy coordinate: the scale follows max |w|
        (1024, 51, 30000, "f64", False),
        (1024, 512, 3000, "f32", False),  # m/p = 1/2: beyond the banded path's shared memory
        (2048, 256, 4000, "f32", False),
        (256, 25, 3, "f32", False),  # fewer rows than one chunk
    ],
)
def test_tc_matches_oracle(skc, monkeypatch, p, m, n, compute, outlier):
    sk = _sketch(skc, p, m, n, p + m + n, compute, outlier)
    monkeypatch.setenv("SKC_COV_PATH", "tc")
    C = skc.estimate_covariance(sk).matrix
    assert rel_fro(C, _oracle(sk, p)) < 1e-5


def test_tc_agrees_with_band_and_is_deterministic(skc, monkeypatch):
    sk = _sketch(skc, 512, 48, 40000, 9)
    monkeypatch.setenv("SKC_COV_PATH", "band")
    Cb = skc.estimate_covariance(sk).matrix
    monkeypatch.setenv("SKC_COV_PATH", "tc")
    Ct = skc.estimate_covariance(sk).matrix
    assert rel_fro(Ct, Cb) < 1e-5
    assert np.array_equal(Ct, skc.estimate_covariance(sk).matrix)  # same launch shape: same bits


def test_tc_short_windows(skc, monkeypatch):
    # one-chunk accumulation windows: every chunk is drained from TMEM (exercises the
    # double-buffered accumulator hand-off); shorter windows truncate less
    sk = _sketch(skc, 256, 40, 9000, 4)
    monkeypatch.setenv("SKC_COV_PATH", "tc")
    C1 = skc.estimate_covariance(sk).matrix
    monkeypatch.setenv("SKC_COVTC_WINDOW", "1")
    C2 = skc.estimate_covariance(sk).matrix
    e1, e2 = rel_fro(C1, _oracle(sk, 256)), rel_fro(C2, _oracle(sk, 256))
    assert e2 < 1e-6 and e2 < e1 < 1e-5


def test_tc_default_for_large_m(skc):
    # no override: m above the measured crossover takes the tensor cores, and m/p = 1/2
    # works at all (the banded path has no room for it)
    sk = _sketch(skc, 512, 256, 2000, 21)
    C = skc.estimate_covariance(sk).matrix
    assert rel_fro(C, _oracle(sk, 512)) < 1e-5
