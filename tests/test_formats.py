"""DNSE1 / SKCH1 formats and the out-of-core dense source.

Golden bytes come from the reference's own writers (tests/golden/make_golden.py formats).
Host-side DNSE1 tests run on CPU. SKCH1 goes through the GPU pack / unpack kernels, and
those tests are marked gpu: files written here must equal the reference's bytes exactly,
because the fp64 sketch is bit-identical to the reference's.
"""

import numpy as np
import pytest
import torch

from paper_1511_00152_b200 import io as skio
from paper_1511_00152_b200.errors import DimensionError, ParameterError


def _case(golden, name):
    g = golden("formats")
    p, n, ss, ms = (int(v) for v in g[f"{name}_meta"])
    return g, g[f"{name}_X"], str(g[f"{name}_kind"]), p, n, ss, ms, float(g[f"{name}_gamma"])


@pytest.mark.parametrize("name", ["had", "none", "had64"])
def test_dense_bytes_match_reference(golden, tmp_path, name):
    g, X, *_ = _case(golden, name)
    path = tmp_path / "m.dnse"
    skio.write_dense(path, X)
    assert path.read_bytes() == g[f"{name}_dnse"].tobytes()
    ref = tmp_path / "ref.dnse"
    ref.write_bytes(g[f"{name}_dnse"].tobytes())
    assert np.array_equal(skio.read_dense(ref), X)


def test_dense_magic_and_truncation(tmp_path):
    bad = tmp_path / "bad"
    bad.write_bytes(b"WRONG" + b"\x00" * 32)
    with pytest.raises(DimensionError):
        skio.read_dense(bad)
    with pytest.raises(DimensionError):
        skio.DenseFileSource(bad)
    X = np.ones((4, 6))
    path = tmp_path / "m.dnse"
    skio.write_dense(path, X)
    path.write_bytes(path.read_bytes()[:-16])
    with pytest.raises(DimensionError):
        skio.read_dense(path)
    src = skio.DenseFileSource(path, chunk_cols=3)
    with pytest.raises(DimensionError, match="column offset 3"):
        np.hstack(list(src.chunks()))
    with pytest.raises(DimensionError):
        skio.write_dense(tmp_path / "v.dnse", np.ones(3))
    with pytest.raises(ParameterError):
        skio.DenseFileSource(path, chunk_cols=0)


def test_dense_file_source_chunks_and_passes(tmp_path):
    X = np.random.default_rng(1).standard_normal((5, 23))
    path = tmp_path / "m.dnse"
    skio.write_dense(path, X)
    src = skio.DenseFileSource(path, chunk_cols=4)
    assert (src.p, src.n) == (5, 23)
    blocks = list(src.chunks())
    assert [b.shape[1] for b in blocks] == [4, 4, 4, 4, 4, 3]
    assert np.array_equal(np.hstack(blocks), X)
    assert src.passes == 1
    rows = [np.asarray(r) for r in src.row_chunks()]
    assert np.array_equal(np.vstack(rows), X.T)
    assert src.passes == 2


# ------------------------------------------------------------------ GPU (SKCH1)
@pytest.fixture(scope="module")
def skc():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_1511_00152_b200 as skc

    return skc


@pytest.mark.gpu
@pytest.mark.parametrize("name", ["had", "none", "had64"])
def test_sketch_file_bytes_match_reference(skc, golden, tmp_path, name):
    g, X, kind, p, n, ss, ms, gamma = _case(golden, name)
    spec = skc.PreconditionSpec.create(kind, p, sign_seed=ss)
    plan = skc.plan_for(spec, gamma, master_seed=ms)
    sk = skc.sketch_stream(X, spec, plan, compute="f64")
    path = tmp_path / "s.skch"
    skio.write_sketch(path, sk)
    assert path.read_bytes() == g[f"{name}_skch"].tobytes()
    ref = tmp_path / "ref.skch"
    ref.write_bytes(g[f"{name}_skch"].tobytes())
    back = skio.read_sketch(ref)
    assert back.spec == spec and back.plan == plan and back.n == n
    assert torch.equal(back.indices, sk.indices)
    assert back.values.cpu().numpy().tobytes() == sk.values.cpu().numpy().tobytes()


@pytest.mark.gpu
def test_sketch_file_large_chunks_and_errors(skc, tmp_path, monkeypatch):
    # several pack / unpack chunks, fp32 values widened exactly to f64
    monkeypatch.setattr(skio, "RECORD_CHUNK", 1000)
    rng = np.random.default_rng(9)
    X = rng.standard_normal((128, 3500)).astype(np.float32)
    spec = skc.PreconditionSpec.create("hadamard", 128, sign_seed=4)
    plan = skc.plan_for(spec, 0.2, master_seed=8)
    sk = skc.sketch_stream(X, spec, plan, compute="f32")
    path = tmp_path / "s.skch"
    skio.write_sketch(path, sk)
    assert path.stat().st_size == 61 + 3500 * 12 * plan.m
    back = skio.read_sketch(path)
    assert torch.equal(back.indices, sk.indices)
    assert torch.equal(back.values, sk.values.to(torch.float64))
    path.write_bytes(path.read_bytes()[:-7])
    with pytest.raises(DimensionError, match="truncated"):
        skio.read_sketch(path)
    bad = tmp_path / "bad"
    bad.write_bytes(b"NOTSK" + b"\x00" * 64)
    with pytest.raises(DimensionError):
        skio.read_sketch(bad)


@pytest.mark.gpu
def test_sketch_stream_from_dense_file(skc, tmp_path):
    # out-of-core: pinned chunk reads, copies overlapped with the kernels, same bytes
    rng = np.random.default_rng(10)
    X = rng.standard_normal((200, 1001))
    path = tmp_path / "m.dnse"
    skio.write_dense(path, X)
    spec = skc.PreconditionSpec.create("hadamard", 200, sign_seed=6)
    plan = skc.plan_for(spec, 0.1, master_seed=7)
    src = skio.DenseFileSource(path, chunk_cols=97)
    a = skc.sketch_stream(src, spec, plan, compute="f64")
    b = skc.sketch_stream(X, spec, plan, compute="f64")
    assert src.passes == 1
    assert torch.equal(a.indices, b.indices) and torch.equal(a.values, b.values)
