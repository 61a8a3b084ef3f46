"""Philox sampler (north_star's counter-based alternative) and supplied-index sketching.

The oracle's Philox4x32-10 is pinned to the published known-answer vectors (Salmon et al.
SC'11, the Random123 library). The GPU sampler must equal the oracle bit for bit. Sketching
at supplied indices must equal the fused oracle-mode sketch when given the same indices.
"""

import numpy as np
import pytest
import torch

from oracle import oracle as O


# ------------------------------------------------------------------ oracle (CPU)
@pytest.mark.parametrize("ctr,key,want", [
    ((0, 0, 0, 0), (0, 0), (0x6627E8D5, 0xE169C58D, 0xBC57AC4C, 0x9B00DBD8)),
    ((0xFFFFFFFF,) * 4, (0xFFFFFFFF, 0xFFFFFFFF), (0x408F276D, 0x41C83B0E, 0xA20BC7C6, 0x6D5451FD)),
    ((0x243F6A88, 0x85A308D3, 0x13198A2E, 0x03707344), (0xA4093822, 0x299F31D0),
     (0xD16CFE09, 0x94FDCCEB, 0x5001E420, 0x24126EA1)),
])
def test_philox_known_answers(ctr, key, want):
    assert tuple(int(v) for v in O.philox4x32_10(ctr, key)) == want


def test_philox_sampler_is_uniform_without_replacement():
    n, p, m = 40000, 512, 26
    a = O.philox_indices(11, 0, n, p, m).astype(np.int64)
    assert ((a[:, 1:] - a[:, :-1]) > 0).all() and a.min() >= 0 and a.max() < p
    f = np.bincount(a.ravel(), minlength=p) / n
    sd = np.sqrt(m / p * (1 - m / p) / n)
    assert np.abs(f - m / p).max() < 5.5 * sd  # every coordinate kept with probability m/p
    # pairs are (nearly) independent: P(j and k both kept) = m(m-1) / (p(p-1))
    both = ((a == 3).any(1) & (a == 400).any(1)).mean()
    assert abs(both - m * (m - 1) / (p * (p - 1))) < 6 * np.sqrt(m * m / p / p / n)
    assert np.array_equal(O.philox_indices(3, 5, 9, 64, 64), np.tile(np.arange(64, dtype=np.uint32), (4, 1)))
    assert np.array_equal(O.philox_indices(3, 100, 107, 1000, 9), O.philox_indices(3, 0, 107, 1000, 9)[100:])


def test_plan_sampler_validation():
    from paper_1511_00152_b200 import ParameterError, SamplingPlan

    assert SamplingPlan(1, 8, 3).sampler == "oracle"
    with pytest.raises(ParameterError):
        SamplingPlan(1, 8, 3, sampler="mt19937")


# ------------------------------------------------------------------ GPU
@pytest.fixture(scope="module")
def skc():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_1511_00152_b200 as skc

    return skc


@pytest.mark.gpu
@pytest.mark.parametrize("p,m,col0,n", [(1024, 51, 0, 100000), (4096, 82, 12345, 3000), (512, 26, 7, 5000),
                                        (64, 64, 0, 100), (37, 5, 3, 999), (2048, 1, 0, 2000), (8, 7, 2 ** 33, 50)])
def test_gpu_philox_matches_oracle(skc, p, m, col0, n):
    plan = skc.SamplingPlan(master_seed=2026 + p, p=p, m=m, sampler="philox")
    got = plan.device_indices(col0, col0 + n).cpu().numpy().astype(np.uint32)
    assert np.array_equal(got, O.philox_indices(2026 + p, col0, col0 + n, p, m))


@pytest.mark.gpu
def test_sketch_stream_philox_and_supplied_indices(skc):
    rng = np.random.default_rng(4)
    p, n = 300, 2500
    X = rng.standard_normal((p, n))
    spec = skc.PreconditionSpec.create("hadamard", p, sign_seed=9)
    ph = skc.plan_for(spec, 0.1, master_seed=17, sampler="philox")
    sk = skc.sketch_stream(skc.ArraySource(X, chunk_cols=333), spec, ph, compute="f64")
    idx = O.philox_indices(17, 0, n, spec.p_pad, ph.m)
    assert np.array_equal(sk.host_indices(), idx)
    Y = O.precondition_rows(X.T.copy(), spec.p_pad, O.HADAMARD, 9)
    assert np.array_equal(sk.host_values(), np.take_along_axis(Y, idx.astype(np.int64), axis=1))
    # supplied indices: the oracle-mode sampler's indices reproduce the fused oracle sketch
    orc = skc.plan_for(spec, 0.1, master_seed=17)
    ref = skc.sketch_stream(X, spec, orc, compute="f64")
    given = skc.sketch_stream(X, spec, orc, compute="f64", indices=ref.host_indices())
    assert torch.equal(given.indices, ref.indices) and torch.equal(given.values, ref.values)
    f32 = skc.sketch_stream(X.astype(np.float32), spec, orc, compute="f32", indices=ref.indices)
    assert np.abs(f32.host_values() - ref.host_values()).max() < 2e-6 * np.abs(ref.host_values()).max()
    with pytest.raises(skc.DimensionError):
        skc.sketch_stream(X, spec, orc, indices=ref.host_indices()[:, ::-1].copy())
    with pytest.raises(skc.DimensionError):
        skc.sketch_stream(X, spec, orc, indices=ref.host_indices()[:10])


@pytest.mark.gpu
def test_philox_edges_and_identity_kind(skc):
    for p, m in ((1, 1), (5, 5), (4096, 4096), (3, 1)):
        plan = skc.SamplingPlan(master_seed=p * 31, p=p, m=m, sampler="philox")
        got = plan.device_indices(0, 40).cpu().numpy().astype(np.uint32)
        assert np.array_equal(got, O.philox_indices(p * 31, 0, 40, p, m))
        if m == p:
            assert np.array_equal(got, np.tile(np.arange(p, dtype=np.uint32), (40, 1)))
    # kind "none": values are the raw coordinates at the sampled indices (transform.py:141-146)
    rng = np.random.default_rng(5)
    X = rng.standard_normal((37, 300))
    spec = skc.PreconditionSpec.create("none", 37)
    plan = skc.SamplingPlan(3, 37, 6, sampler="philox")
    sk = skc.sketch_stream(X, spec, plan, compute="f64")
    idx = O.philox_indices(3, 0, 300, 37, 6)
    assert np.array_equal(sk.host_indices(), idx)
    assert np.array_equal(sk.host_values(), np.take_along_axis(X.T, idx.astype(np.int64), axis=1))
