"""K3 covariance kernel A/B at the C3 shape (p=1024, m=51) and C1/C2-like shapes.

Builds a sketch with the Philox sampler and Gaussian f64 values, runs K2 for the fixed-point
statistics, then times skc_cov_accumulate with each kernel variant selected by environment
(SKC_COV_KERNEL=band: the round-1 band kernel) and checks that every variant's triangle is
bit-identical (the fixed-point sums are exact and order-independent).

usage: python tools/k3_ab.py [n_log2=22] [reps=5]
"""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1511_00152_b200 import _lib  # noqa: E402

dev = torch.device("cuda")
L = _lib.lib()
nlog = int(sys.argv[1]) if len(sys.argv) > 1 else 22
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 5
variants = {"old": {"SKC_COV_KERNEL": "band"}, "flat": {"SKC_COV_KERNEL": "flat"}}
shapes = ((1024, 51), (512, 26), (2048, 51), (256, 25))
for p, m in shapes[: int(os.environ.get("K3AB_SHAPES", "4"))]:
    n = 1 << nlog
    g = torch.Generator(device=dev).manual_seed(p + m)
    idx = torch.empty((n, m), dtype=torch.int32, device=dev)
    st = _lib.stream_ptr(dev)
    _lib.call("skc_indices_philox", p + m, 0, n, p, m, idx.data_ptr(), st)
    val = torch.randn((n, m), device=dev, generator=g, dtype=torch.float64) * 1.3
    acc = torch.zeros(p, dtype=torch.float64, device=dev)
    stats = torch.zeros(3, dtype=torch.float64, device=dev)
    ws1 = _lib.workspace(L.skc_moments_workspace(n, m, p), dev)
    _lib.call("skc_moments", idx.data_ptr(), val.data_ptr(), _lib.F64, n, m, p, acc.data_ptr(), stats.data_ptr(),
              ws1.data_ptr(), ws1.numel(), st)
    res = {}
    for name, env in variants.items():
        os.environ.pop("SKC_COV_KERNEL", None)
        os.environ.update(env)
        ws2 = _lib.workspace(L.skc_cov_workspace(n, m, p), dev)  # band count depends on the kernel
        tri = torch.zeros(p * (p + 1) // 2, dtype=torch.float64, device=dev)

        def run():
            tri.zero_()
            _lib.call("skc_cov_accumulate", idx.data_ptr(), val.data_ptr(), _lib.F64, n, m, p, stats.data_ptr(),
                      tri.data_ptr(), ws2.data_ptr(), ws2.numel(), st)

        run()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(reps):
            run()
        e1.record()
        torch.cuda.synchronize()
        res[name] = (e0.elapsed_time(e1) / reps, tri.clone())
    os.environ.pop("SKC_COV_KERNEL", None)
    base = res["old"][1]
    upd = n * m * (m + 1) / 2
    line = " ".join(f"{k} {t:.3f} ms ({upd / t / 1e9:.3f}e12/s) same={torch.equal(tri, base)}"
                    for k, (t, tri) in res.items())
    print(f"p={p} m={m} n=2^{nlog}: {line}", flush=True)
    del idx, val, ws1, ws2
    torch.cuda.empty_cache()
