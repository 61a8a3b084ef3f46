"""Generate golden fixtures by running the REFERENCE implementation.

Run in the build container, where the reference is importable:

    PYTHONPATH=/root/reference/pkg/src python tests/golden/make_golden.py

This writes ``tests/golden/*.npz``. The fixtures are small and committed. The
GPU box has no ``/root/reference``, so every test there reads these files
instead. All inputs are seeded synthetic data. fp32-representable samples are
stored as float32 and upcast exactly to float64 before they are fed to the
reference, which is the same data the GPU path consumes.
"""

from __future__ import annotations

import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
from datagen import digest, mixture, spiked  # noqa: E402

try:
    import sketchpipe as skp
    from sketchpipe import _hash
    from sketchpipe.cluster import _SparseOps
    from sketchpipe.transform import _fwht_axis0
except ImportError:  # pragma: no cover
    sys.exit("reference not importable: set PYTHONPATH=/root/reference/pkg/src")

OUT = os.path.dirname(os.path.abspath(__file__))
SEED = 2026
LAMS = [50.0, 40.0, 30.0, 20.0, 10.0]


def gen_hash():
    d = {}
    zs = np.array([0, 1, 2, 0xDEADBEEF, 2**63, 2**64 - 1], dtype=np.uint64)
    d["mix64_in"] = zs
    d["mix64_out"] = np.array([int(_hash.mix64(z)) for z in zs], dtype=np.uint64)
    seeds = np.array([0, 1, 2026, 0xD5, 2**64 - 1], dtype=np.uint64)
    tags = np.array([0xD5, 0x5A, 0x53494748, 7, 0], dtype=np.uint64)
    d["derive_seed_in"] = np.stack([seeds, tags])
    d["derive_seed_out"] = np.array(
        [_hash.derive_seed(int(s), int(t)) for s, t in zip(seeds, tags)], dtype=np.uint64
    )
    for s, p in [(1, 16), (77, 1024), (123, 64), (0, 4096)]:
        d[f"signs_{s}_{p}"] = _hash.sign_array(s, p)
    d["keys_2_0_4_16"] = _hash.column_keys(2, 0, 4, 16)
    d["keys_99_1000_1003_256"] = _hash.column_keys(99, 1000, 1003, 256)
    cases = [
        (2, 16, 4, 0, 4), (2, 256, 25, 0, 64), (42, 50, 7, 990, 1000), (7, 3, 2, 0, 300),
        (9, 4, 1, 0, 300), (1, 6, 6, 0, 5), (13, 512, 26, 123456, 123520), (5, 1024, 51, 2**33, 2**33 + 40),
        (0x8726ACFD89F696E8, 4096, 82, 0, 16), (11, 2048, 102, 10**7 - 8, 10**7), (3, 64, 63, 0, 64),
        (3, 128, 100, 0, 32), (8, 32, 16, 0, 100),
    ]
    meta = []
    for k, (ms, p, m, i0, i1) in enumerate(cases):
        plan = skp.SamplingPlan(master_seed=ms, p=p, m=m)
        d[f"idx_{k}"] = plan.indices_block(i0, i1)
        meta.append([ms & 0xFFFFFFFFFFFFFFFF, p, m, i0, i1])
    d["idx_meta"] = np.array(meta, dtype=np.uint64)
    return d


def gen_transform():
    d = {}
    d["fwht_2"] = skp.fwht_inplace(np.array([1.0, 0.0]))
    d["fwht_4"] = skp.fwht_inplace(np.array([1.0, 1.0, 1.0, 1.0]))
    H = np.column_stack([_fwht_axis0(np.eye(16)[:, [j]].copy()).ravel() for j in range(16)])
    d["hadamard_16"] = H
    rng = np.random.default_rng(SEED)
    meta = []
    for k, (kind, p, seed) in enumerate(
        [("hadamard", 30, 9), ("hadamard", 64, 5), ("hadamard", 100, 11), ("none", 40, 0), ("hadamard", 1024, 77),
         ("hadamard", 4096, 3), ("hadamard", 1, 4), ("hadamard", 2, 4)]
    ):
        spec = skp.PreconditionSpec.create(kind, p, sign_seed=seed)
        X = rng.standard_normal((p, 7)).astype(np.float32)
        d[f"pre_X_{k}"] = X
        d[f"pre_Y_{k}"] = skp.precondition_columns(X.astype(np.float64), spec)
        d[f"unpre_{k}"] = skp.unprecondition_columns(d[f"pre_Y_{k}"], spec)
        meta.append([0 if kind == "hadamard" else 2, p, spec.p_pad, seed])
    d["pre_meta"] = np.array(meta, dtype=np.int64)
    return d


def gen_sketch():
    """sketch_stream + estimators on seeded data; hot-path configs at small n."""
    d = {}
    cases = [
        # name, kind, p, n, gamma, sign_seed, master_seed, pcs
        ("c1", "hadamard", 256, 2000, 25 / 256, 0xCE1A6B4D43BD6E9D, 0x8726ACFD89F696E8, 5),
        ("c3", "hadamard", 1024, 400, 51 / 1024, 11, 12, 3),
        ("c4", "hadamard", 4096, 48, 82 / 4096, 21, 22, 2),
        ("odd", "hadamard", 50, 1000, 0.25, 2, 6, 2),
        ("none", "none", 20, 300, 0.4, 0, 9, 2),
        ("full", "hadamard", 8, 30, 1.0, 2, 8, 2),
        ("tiny", "hadamard", 3, 50, 0.5, 1, 1, 1),
        ("p32", "hadamard", 32, 200, 0.5, 3, 4, 2),
        ("c5", "hadamard", 2048, 96, 102 / 2048, 5, 6, 2),
        ("c2", "hadamard", 512, 1000, 26 / 512, 7, 8, 2),
    ]
    names = []
    for name, kind, p, n, gamma, ss, ms, k in cases:
        spec = skp.PreconditionSpec.create(kind, p, sign_seed=ss)
        plan = skp.plan_for(spec, gamma, master_seed=ms)
        X = spiked(SEED + p + n, p, n, LAMS[: max(1, min(5, p - 1))])
        if name == "odd":
            X[:, 17] = 0.0  # a zero sample keeps m slots
        sk = skp.sketch_stream(skp.ArraySource(X.astype(np.float64), chunk_cols=97), spec, plan)
        d[f"{name}_X_sha"] = np.array(digest(X))
        d[f"{name}_idx"] = sk.indices
        d[f"{name}_val"] = sk.values
        d[f"{name}_mean"] = skp.estimate_mean(sk)
        if plan.m >= 2:
            C = skp.estimate_covariance(sk).matrix
            if spec.p_pad <= 256:
                d[f"{name}_cov"] = C
            else:
                # large p: diagonal, Frobenius norm and a seeded entry subset
                sel = np.random.default_rng(spec.p_pad).integers(0, spec.p_pad, (2, 4096))
                d[f"{name}_cov_diag"] = C.diagonal().copy()
                d[f"{name}_cov_fro"] = np.array(np.linalg.norm(C))
                d[f"{name}_cov_sel"] = sel
                d[f"{name}_cov_selval"] = C[sel[0], sel[1]]
            d[f"{name}_pcs"] = skp.principal_components(sk, k)
        d[f"{name}_meta"] = np.array(
            [0 if kind == "hadamard" else 2, p, spec.p_pad, n, plan.m, ss, ms, k], dtype=np.uint64
        )
        names.append(name)
    d["names"] = np.array(names)
    return d


def gen_kmeans():
    """Lloyd trajectories of the reference's _SparseOps from seeded initial points."""
    d = {}
    rng = np.random.default_rng(SEED + 2)
    cases = [
        ("c2", 512, 3000, 10, 26, 20),
        ("c5", 2048, 600, 20, 102, 10),
        ("small", 64, 800, 5, 7, 30),
        ("empty", 16, 60, 6, 4, 15),
    ]
    names = []
    for name, p, n, K, m, max_iter in cases:
        X = mixture(SEED + p + K, p, n, K, 2.0 if name != "empty" else 0.3)
        spec = skp.PreconditionSpec.create("hadamard", p, sign_seed=SEED + K)
        plan = skp.SamplingPlan(master_seed=SEED * 3 + K, p=spec.p_pad, m=m)
        sk = skp.sketch_stream(X.astype(np.float64), spec, plan)
        ops = _SparseOps(sk)
        chosen = rng.choice(n, K, replace=False)
        if name == "empty":
            chosen[1] = chosen[0]  # duplicate centers force an empty cluster and a reseed
        mu = ops.init_centers(list(chosen))
        prev = None
        labs, mus, cnts, traj, d2s, empties = [], [], [], [], [], []
        for _ in range(max_iter):
            labels, d2min = ops.assign(mu)
            traj.append(float(d2min.sum()))
            labs.append(labels)
            d2s.append(d2min)
            if prev is not None and np.array_equal(labels, prev):
                break
            prev = labels
            mu, empty = ops.update(labels, mu, K)
            for kk in np.flatnonzero(empty):
                ops.reseed(mu, kk, d2min)
            mus.append(mu.copy())
            cnts.append(ops.last_counts.copy())
            empties.append(empty.copy())
        d[f"{name}_X_sha"] = np.array(digest(X))
        d[f"{name}_idx_sha"] = np.array(digest(sk.indices))
        d[f"{name}_val_sha"] = np.array(digest(sk.values))
        d[f"{name}_chosen"] = chosen
        d[f"{name}_labels"] = np.stack(labs).astype(np.int16)
        d[f"{name}_d2min_first"] = d2s[0]
        d[f"{name}_d2min_last"] = d2s[-1]
        if p <= 64:
            d[f"{name}_mu"] = np.stack(mus)
            d[f"{name}_counts"] = np.stack(cnts)
        d[f"{name}_mu_final"] = mus[-1]
        d[f"{name}_counts_final"] = cnts[-1]
        d[f"{name}_empty"] = np.stack(empties)
        d[f"{name}_traj"] = np.array(traj)
        d[f"{name}_final_centers"] = skp.unprecondition_columns(mu, spec)[:p]
        d[f"{name}_meta"] = np.array([p, spec.p_pad, n, K, m, max_iter, SEED + K, SEED * 3 + K], dtype=np.int64)
        names.append(name)
    d["names"] = np.array(names)
    return d


def gen_formats():
    """SKCH1 / DNSE1 bytes written by the reference (io.py) for small seeded inputs."""
    import tempfile

    d = {}
    cases = [("had", "hadamard", 20, 15, 1234, 0.3, 987, 2), ("none", "none", 13, 9, 0, 0.5, 31, 3),
             ("had64", "hadamard", 64, 40, 77, 0.25, 5, 4)]
    with tempfile.TemporaryDirectory() as tmp:
        for name, kind, p, n, ss, gamma, ms, xseed in cases:
            X = np.random.default_rng(xseed).standard_normal((p, n))
            spec = skp.PreconditionSpec.create(kind, p, sign_seed=ss)
            plan = skp.plan_for(spec, gamma, master_seed=ms)
            sk = skp.sketch_stream(X, spec, plan)
            f = os.path.join(tmp, name + ".skch")
            skp.write_sketch(f, sk)
            d[f"{name}_X"] = X
            d[f"{name}_meta"] = np.array([p, n, ss, ms], dtype=np.int64)
            d[f"{name}_gamma"] = np.float64(gamma)
            d[f"{name}_kind"] = np.array(kind)
            d[f"{name}_skch"] = np.frombuffer(open(f, "rb").read(), dtype=np.uint8)
            g = os.path.join(tmp, name + ".dnse")
            skp.write_dense(g, X)
            d[f"{name}_dnse"] = np.frombuffer(open(g, "rb").read(), dtype=np.uint8)
    d["names"] = np.array([c[0] for c in cases])
    return d


def gen_twopass():
    """Reference sparsified_kmeans_two_pass (cluster.py:407-456) on seeded mixtures."""
    d = {}
    cases = [  # name, p, n, K, scale, gamma, n_init, seed, kind, chunk, max_iter
        ("sep", 24, 400, 3, 4.0, 0.3, 3, 19, "hadamard", 100, 100),
        ("mid", 64, 2000, 5, 1.0, 0.2, 2, 3, "hadamard", 512, 50),
        ("none", 16, 150, 3, 3.0, 1.0, 3, 23, "none", 40, 100),
        ("big", 200, 5000, 8, 1.5, 0.1, 2, 7, "hadamard", 1500, 30),
    ]
    for name, p, n, K, scale, gamma, n_init, seed, kind, chunk, max_iter in cases:
        X = mixture(SEED + 17 * p + K, p, n, K, scale).astype(np.float64)
        src = skp.ArraySource(X, chunk_cols=chunk)
        res = skp.sparsified_kmeans_two_pass(src, K, gamma, max_iter=max_iter, n_init=n_init, seed=seed, kind=kind,
                                             chunk_cols=chunk)
        first = skp.sparsified_kmeans(X, K, gamma, max_iter=max_iter, n_init=n_init, seed=seed, kind=kind,
                                      chunk_cols=chunk)
        d[f"{name}_X_sha"] = np.array(digest(X))
        d[f"{name}_cfg"] = np.array([p, n, K, n_init, seed, chunk, max_iter], dtype=np.int64)
        d[f"{name}_f"] = np.array([scale, gamma], dtype=np.float64)
        d[f"{name}_kind"] = np.array(kind)
        d[f"{name}_labels"] = res.assignments.labels.astype(np.int32)
        d[f"{name}_centers"] = res.centers.centers
        d[f"{name}_objective"] = np.float64(res.objective)
        d[f"{name}_first_labels"] = first.assignments.labels.astype(np.int32)
        d[f"{name}_first_centers"] = first.centers.centers
        d[f"{name}_first_objective"] = np.float64(first.objective)
    d["names"] = np.array([c[0] for c in cases])
    return d


GENERATORS = {"hash": gen_hash, "transform": gen_transform, "sketch": gen_sketch, "kmeans": gen_kmeans,
              "formats": gen_formats, "twopass": gen_twopass}


def main():
    which = sys.argv[1:] or list(GENERATORS)
    for fname in which:
        fn = GENERATORS[fname]
        path = os.path.join(OUT, f"{fname}.npz")
        np.savez_compressed(path, **fn())
        print(f"wrote {path} ({os.path.getsize(path) / 1e3:.0f} kB)")


if __name__ == "__main__":
    main()
