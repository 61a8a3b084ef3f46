"""CPU tests: the C ABI library loads and exports every entry point that
include/sketchcu.h declares (no compute calls without a GPU), and the host-side
logic (spec and plan validation, seeds, sharding) mirrors the reference."""

import os
import re

import numpy as np
import pytest
import torch

from oracle import oracle as O

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def header_symbols():
    text = open(os.path.join(ROOT, "include", "sketchcu.h")).read()
    return sorted(set(re.findall(r"\b(skc_[a-z0-9_]+)\s*\(", text)))


@pytest.fixture(scope="module")
def lib():
    from paper_1511_00152_b200 import _build, _lib

    if not os.path.exists(_lib.SO_PATH):
        _build.build()
    return _lib.load_library()


def test_header_declares_the_expected_surface():
    syms = header_symbols()
    for name in ["skc_sketch", "skc_indices", "skc_moments", "skc_cov_accumulate", "skc_cov_finalize",
                 "skc_mean_finalize", "skc_kmeans_assign", "skc_kmeans_partials", "skc_kmeans_centers",
                 "skc_kmeans_reseed", "skc_unprecondition", "skc_precondition", "skc_signs", "skc_fwht"]:
        assert name in syms


def test_library_exports_every_header_symbol(lib):
    from paper_1511_00152_b200 import _lib

    for name in header_symbols():
        assert hasattr(lib, name), f"{name} declared in sketchcu.h but not exported"
        assert name in _lib.SIGNATURES, f"{name} has no ctypes signature"
    assert lib.skc_abi_version() == 1
    assert lib.skc_max_p_pad() == 4096


def test_workspace_queries_are_host_only(lib):
    # size queries never touch the device
    assert lib.skc_cov_workspace(1 << 20, 51, 1024) > 0
    assert lib.skc_moments_workspace(1 << 20, 51, 1024) > 0
    assert lib.skc_kmeans_partials_workspace(200000, 26, 512, 10) > 0
    assert lib.skc_kmeans_assign_workspace(200000, 512, 10) >= 2 * 512 * 10 * 8


def test_product_path_fails_loudly_without_gpu():
    import paper_1511_00152_b200 as skc

    if torch.cuda.is_available():
        pytest.skip("a GPU is present")
    spec = skc.PreconditionSpec.create("hadamard", 16, 1)
    with pytest.raises(skc.DeviceError):
        skc.sketch_stream(np.zeros((16, 4), np.float32), spec, skc.SamplingPlan(1, 16, 4))


def test_spec_and_plan_validation_mirror_reference():
    import paper_1511_00152_b200 as skc

    with pytest.raises(skc.ParameterError):
        skc.PreconditionSpec.create("fourier", 8)
    with pytest.raises(skc.DimensionError):
        skc.PreconditionSpec(kind="hadamard", sign_seed=0, p=5, p_pad=6)
    with pytest.raises(skc.DimensionError):
        skc.PreconditionSpec(kind="dct", sign_seed=0, p=5, p_pad=8)
    assert skc.PreconditionSpec.create("hadamard", 5).p_pad == 8
    assert skc.PreconditionSpec.create("hadamard", 8).eta == 1.0
    assert skc.PreconditionSpec.create("dct", 8).eta == 0.5
    with pytest.raises(skc.ParameterError):
        _ = skc.PreconditionSpec.create("none", 8).eta
    with pytest.raises(skc.ParameterError):
        skc.SamplingPlan(master_seed=0, p=4, m=0)
    with pytest.raises(skc.ParameterError):
        skc.SamplingPlan(master_seed=0, p=4, m=5)
    assert skc.SamplingPlan(master_seed=0, p=4, m=2).gamma == 0.5
    spec = skc.PreconditionSpec.create("hadamard", 100)
    assert skc.plan_for(spec, 0.3, 1).m == round(0.3 * 128)
    for bad in (0.0, 1.5):
        with pytest.raises(skc.ParameterError):
            skc.plan_for(spec, bad, 1)
    with pytest.raises(skc.ParameterError):
        skc.plan_for(skc.PreconditionSpec.create("none", 200), 0.001, 1)
    assert [skc.next_pow2(x) for x in (1, 2, 3, 512, 513)] == [1, 2, 4, 512, 1024]


def test_run_seeds_match_reference_derivation():
    from paper_1511_00152_b200.cluster import derive_seed

    for s in (0, 1, 2026, 2**64 - 1, 12345678901234):
        for tag in (0xD5, 0x5A):
            assert derive_seed(s, tag) == O.derive_seed(s, tag)


def test_shard_bounds_and_owner():
    from paper_1511_00152_b200 import dist

    for n in (1, 7, 1000, 16777216, 10_000_000):
        for w in (1, 2, 3, 8):
            bounds = [dist.shard_bounds(n, r, w) for r in range(w)]
            assert bounds[0][0] == 0 and bounds[-1][1] == n
            assert all(bounds[r][1] == bounds[r + 1][0] for r in range(w - 1))
            for i in {0, n - 1, n // 2, n // 3}:
                r = dist.owner_of(i, n, w)
                assert bounds[r][0] <= i < bounds[r][1]


def test_count_diagonal_helpers():
    from paper_1511_00152_b200 import CountDiagonal

    counts = np.array([[2, 0], [2, 0], [1, 0], [1, 0]])
    cd = CountDiagonal(counts=counts)
    assert cd.cluster_sizes(2).tolist() == [3, 0]
    dev = cd.hk_deviations(2)
    assert np.isclose(dev[0], np.abs(4 * counts[:, 0] / (2 * 3) - 1).max()) and np.isnan(dev[1])
