"""K1b TMA-staged gather (gather.cu): the values of sketch_stream (sketch.py:211-220) for fp32
rows at every p the kernel is instantiated for, ragged n, strided rows, both compute types.

compute="f64" must equal the reference arithmetic bit for bit (oracle restatement of
transform.py:92-110 on the exact fp64 upcast of the fp32 rows); compute="f32" must equal the
same butterfly order evaluated in IEEE fp32 (numpy float32 below), also bit for bit.
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


def precondition_f32(X: np.ndarray, p: int, sign_seed: int) -> np.ndarray:
    """transform.py:180-189 evaluated in IEEE fp32 in the reference stage order."""
    n = X.shape[0]
    a = X.astype(np.float32) * O.signs(sign_seed, p).astype(np.float32)[None, :]
    h = 1
    while h < p:
        b = a.reshape(n, p // (2 * h), 2, h)
        x, y = b[:, :, 0, :].copy(), b[:, :, 1, :].copy()
        a = np.stack([x + y, x - y], axis=2).reshape(n, p)
        h *= 2
    return a * np.float32(1.0 / np.sqrt(p))


def run_given(skc, rows: torch.Tensor, p: int, m: int, compute: str, ss=5, ms=6):
    from paper_1511_00152_b200 import _lib

    n = rows.shape[0]
    idx = torch.empty((n, m), dtype=torch.int32, device=rows.device)
    vdt = torch.float64 if compute == "f64" else torch.float32
    val = torch.empty((n, m), dtype=vdt, device=rows.device)
    st = _lib.stream_ptr(rows.device)
    _lib.call("skc_indices", ms, 0, n, p, m, idx.data_ptr(), st)
    _lib.call("skc_sketch_given", rows.data_ptr(), _lib.F32, rows.stride(0), n, p, p, 0, ss, m,
              _lib.F64 if compute == "f64" else _lib.F32, idx.data_ptr(), val.data_ptr(),
              _lib.F64 if compute == "f64" else _lib.F32, st)
    torch.cuda.synchronize()
    return idx.cpu().numpy().astype(np.int64), val.cpu().numpy()


@pytest.mark.parametrize("p", [32, 64, 128, 256, 512, 1024, 2048, 4096])
@pytest.mark.parametrize("compute", ["f64", "f32"])
def test_gather_bit_exact_every_p(skc, p, compute):
    rng = np.random.default_rng(p)
    n = 1037 if p <= 1024 else 203  # ragged: not a multiple of any tile
    m = max(2, p // 20)
    X = (rng.standard_normal((n, p)) * np.exp(rng.uniform(-3, 3, (n, 1)))).astype(np.float32)
    X[5] = 0.0
    idx, val = run_given(skc, torch.as_tensor(X).cuda(), p, m, compute)
    assert np.array_equal(idx.astype(np.uint32), O.indices_block(6, 0, n, p, m))
    if compute == "f64":
        Y = O.precondition_rows(X.astype(np.float64), p, O.HADAMARD, 5)
    else:
        Y = precondition_f32(X, p, 5)
    assert np.array_equal(val, np.take_along_axis(Y, idx, axis=1))


@pytest.mark.parametrize("extra", [4, 1])
def test_gather_strided_rows(skc, extra):
    # ld = p + 4 keeps 16-byte rows (TMA path); ld = p + 1 takes the cp.async fallback
    p, n, m = 1024, 300, 51
    rng = np.random.default_rng(7)
    W = rng.standard_normal((n, p + extra)).astype(np.float32)
    Xd = torch.as_tensor(W).cuda()[:, :p]
    idx, val = run_given(skc, Xd, p, m, "f64")
    Y = O.precondition_rows(W[:, :p].astype(np.float64), p, O.HADAMARD, 5)
    assert np.array_equal(val, np.take_along_axis(Y, idx, axis=1))


@pytest.mark.parametrize("n", [1, 2, 9])
def test_gather_tiny_n(skc, n):
    p, m = 2048, 102
    X = np.random.default_rng(n).standard_normal((n, p)).astype(np.float32)
    idx, val = run_given(skc, torch.as_tensor(X).cuda(), p, m, "f64")
    Y = O.precondition_rows(X.astype(np.float64), p, O.HADAMARD, 5)
    assert np.array_equal(val, np.take_along_axis(Y, idx, axis=1))


def test_sketch_stream_default_uses_bit_exact_values(skc):
    # the drop-in call on fp32 device rows: indices + fp64 values equal the oracle's
    p, n, m = 1024, 5000, 51
    X = np.random.default_rng(11).standard_normal((n, p)).astype(np.float32)
    spec = skc.PreconditionSpec.create("hadamard", p, sign_seed=3)
    plan = skc.SamplingPlan(4, p, m)
    sk = skc.sketch_stream(skc.RowSource(torch.as_tensor(X).cuda()), spec, plan)
    io, vo = O.sketch(X, p, O.HADAMARD, 3, 4, m, nthreads=4)
    assert sk.values.dtype == torch.float64
    assert np.array_equal(sk.host_indices(), io) and np.array_equal(sk.host_values(), vo)
