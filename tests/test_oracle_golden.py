"""Pin the CPU oracle to the reference's own outputs (tests/golden, made by
tests/golden/make_golden.py from /root/reference). Bit-exact everywhere: integer
hashing, indices and counts, and the fp64 transform, estimators and K-means
arithmetic, which run in the reference's operation order."""

import numpy as np
import pytest

from datagen import digest, mixture, spiked
from oracle import oracle as O

LAMS = [50.0, 40.0, 30.0, 20.0, 10.0]
SEED = 2026


def test_hash_streams(golden):
    g = golden("hash")
    for z, want in zip(g["mix64_in"], g["mix64_out"]):
        assert O.mix64(int(z)) == int(want)
    for s, t, want in zip(g["derive_seed_in"][0], g["derive_seed_in"][1], g["derive_seed_out"]):
        assert O.derive_seed(int(s), int(t)) == int(want)
    for s, p in [(1, 16), (77, 1024), (123, 64), (0, 4096)]:
        assert np.array_equal(O.signs(s, p), g[f"signs_{s}_{p}"])
    assert np.array_equal(O.column_keys(2, 0, 4, 16), g["keys_2_0_4_16"])
    assert np.array_equal(O.column_keys(99, 1000, 1003, 256), g["keys_99_1000_1003_256"])


def test_known_answers_from_survey():
    # SURVEY.md 8(c) known-answer values (computed from the reference)
    assert O.mix64(1) == 0x5692161D100B05E5
    assert O.derive_seed(2026, 0xD5) == 0xCE1A6B4D43BD6E9D
    assert O.derive_seed(2026, 0x5A) == 0x8726ACFD89F696E8
    assert O.signs(1, 16).tolist() == [-1, 1, -1, -1, 1, 1, -1, 1, -1, -1, 1, -1, 1, 1, 1, -1]
    assert O.indices_block(2, 0, 4, 16, 4).tolist() == [[3, 7, 11, 15], [0, 2, 11, 13], [4, 5, 7, 8], [3, 12, 13, 15]]
    assert O.indices_block(2, 0, 1, 256, 25)[0].tolist() == [
        25, 27, 30, 48, 52, 64, 85, 114, 118, 121, 128, 139, 140, 146, 168, 189, 200, 214, 218, 223, 231, 235, 238,
        249, 254]


def test_indices_blocks(golden):
    g = golden("hash")
    for k, (ms, p, m, i0, i1) in enumerate(g["idx_meta"]):
        got = O.indices_block(int(ms), int(i0), int(i1), int(p), int(m))
        assert np.array_equal(got, g[f"idx_{k}"]), (ms, p, m, i0, i1)


def test_fwht_known_answers(golden):
    g = golden("transform")
    assert np.array_equal(O.fwht([1.0, 0.0]), g["fwht_2"])
    assert np.array_equal(O.fwht([1.0, 1.0, 1.0, 1.0]), g["fwht_4"])
    H = np.column_stack([O.fwht(np.eye(16)[:, j]) for j in range(16)])
    assert np.array_equal(H, g["hadamard_16"])


def test_precondition_bit_exact(golden):
    g = golden("transform")
    for k, (kind, p, p_pad, seed) in enumerate(g["pre_meta"]):
        X = g[f"pre_X_{k}"]
        Y = O.precondition_rows(X.T.astype(np.float64), int(p_pad), int(kind), int(seed))
        assert np.array_equal(Y.T, g[f"pre_Y_{k}"]), (kind, p)
        B = O.unprecondition_rows(g[f"pre_Y_{k}"].T, int(kind), int(seed))
        assert np.array_equal(B.T, g[f"unpre_{k}"])


def _sketch_case(g, name):
    kind, p, p_pad, n, m, ss, ms, k = (int(v) for v in g[f"{name}_meta"])
    X = spiked(SEED + p + n, p, n, LAMS[: max(1, min(5, p - 1))])
    if name == "odd":
        X[:, 17] = 0.0
    assert digest(X) == str(g[f"{name}_X_sha"])
    return X, kind, p, p_pad, n, m, ss, ms, k


@pytest.mark.parametrize("name", ["c1", "c3", "c4", "odd", "none", "full", "tiny", "p32", "c5", "c2"])
def test_sketch_and_estimators_bit_exact(golden, name):
    g = golden("sketch")
    X, kind, p, p_pad, n, m, ss, ms, k = _sketch_case(g, name)
    idx, val = O.sketch(X.T.copy(), p_pad, kind, ss, ms, m, nthreads=4)
    assert np.array_equal(idx, g[f"{name}_idx"])
    assert np.array_equal(val, g[f"{name}_val"])
    assert np.array_equal(O.estimate_mean(idx, val, p, p_pad, kind, ss), g[f"{name}_mean"])
    if m >= 2:
        C = O.estimate_covariance(idx, val, p_pad)
        if f"{name}_cov" in g:
            assert np.array_equal(C, g[f"{name}_cov"])
        else:
            sel = g[f"{name}_cov_sel"]
            assert np.array_equal(C.diagonal(), g[f"{name}_cov_diag"])
            assert np.array_equal(C[sel[0], sel[1]], g[f"{name}_cov_selval"])
        U = O.principal_components(idx, val, p, p_pad, kind, ss, k)
        ref = g[f"{name}_pcs"]
        # eigenvector signs are arbitrary (parity-unpinned): align signs, then compare
        sgn = np.sign(np.sum(U * ref, axis=0))
        assert np.abs(U * sgn - ref).max() < 1e-8


@pytest.mark.parametrize("name", ["c2", "c5", "small", "empty"])
def test_kmeans_trajectory_bit_exact(golden, name):
    g = golden("kmeans")
    p, p_pad, n, K, m, max_iter, ss, ms = (int(v) for v in g[f"{name}_meta"])
    X = mixture(SEED + p + K, p, n, K, 2.0 if name != "empty" else 0.3)
    assert digest(X) == str(g[f"{name}_X_sha"])
    idx, val = O.sketch(X.T.copy(), p_pad, O.HADAMARD, ss, ms, m, nthreads=4)
    assert digest(idx) == str(g[f"{name}_idx_sha"]) and digest(val) == str(g[f"{name}_val_sha"])
    mu0 = O.init_centers(idx, val, g[f"{name}_chosen"], p_pad)
    labels, mu, traj, iters = O.lloyd(idx, val, mu0, max_iter)
    assert iters == g[f"{name}_labels"].shape[0]
    assert np.array_equal(labels, g[f"{name}_labels"][-1])
    assert traj == g[f"{name}_traj"].tolist()
    assert np.array_equal(mu, g[f"{name}_mu_final"])
    _, counts, _ = O.kmeans_update(idx, val, g[f"{name}_labels"][-2], g[f"{name}_mu"][-2] if f"{name}_mu" in g
                                   else mu0)
    assert np.array_equal(counts, g[f"{name}_counts_final"])
    assert np.array_equal(O.kmeans_assign(idx, val, mu0)[1], g[f"{name}_d2min_first"])


def test_pairwise_sum_matches_numpy():
    rng = np.random.default_rng(0)
    for n in [1, 5, 8, 9, 51, 128, 129, 1000, 12345]:
        a = rng.standard_normal(n)
        assert O.pairwise_sum(a) == a.sum()
