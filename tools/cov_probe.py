"""K3 covariance paths on synthetic sketches: banded shared memory vs L2-resident global atomics.

usage: SKC_COV_PATH=b|g python tools/cov_probe.py   (each config also checked against the other path)
"""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1511_00152_b200 import _lib  # noqa: E402

dev = torch.device("cuda")
L = _lib.lib()
for p, m, n in ((1024, 51, 1 << 22), (2048, 102, 1 << 21), (2048, 51, 1 << 22), (4096, 82, 1 << 21), (256, 25, 1 << 22)):
    g = torch.Generator(device=dev).manual_seed(p + m)
    idx = torch.empty((n, m), dtype=torch.int32, device=dev)
    _lib.call("skc_indices_philox", p + m, 0, n, p, m, idx.data_ptr(), _lib.stream_ptr(dev))
    val = torch.randn((n, m), device=dev, generator=g, dtype=torch.float32)
    acc = torch.zeros(p, dtype=torch.float64, device=dev)
    stats = torch.zeros(3, dtype=torch.float64, device=dev)
    ws1 = _lib.workspace(L.skc_moments_workspace(n, m, p), dev)
    st = _lib.stream_ptr(dev)
    _lib.call("skc_moments", idx.data_ptr(), val.data_ptr(), _lib.F32, n, m, p, acc.data_ptr(), stats.data_ptr(),
              ws1.data_ptr(), ws1.numel(), st)
    ws2 = _lib.workspace(L.skc_cov_workspace(n, m, p), dev)
    res = {}
    for path in ("b", "g"):
        os.environ["SKC_COV_PATH"] = path
        tri = torch.zeros(p * (p + 1) // 2, dtype=torch.float64, device=dev)

        def run():
            tri.zero_()
            _lib.call("skc_cov_accumulate", idx.data_ptr(), val.data_ptr(), _lib.F32, n, m, p, stats.data_ptr(),
                      tri.data_ptr(), ws2.data_ptr(), ws2.numel(), st)

        run()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(3):
            run()
        e1.record()
        torch.cuda.synchronize()
        res[path] = (e0.elapsed_time(e1) / 3, tri.clone())
    same = torch.equal(res["b"][1], res["g"][1])
    upd = n * m * (m + 1) / 2
    print(f"p={p} m={m} n={n}: banded {res['b'][0]:.2f} ms ({upd / res['b'][0] / 1e9:.2f}e12/s), "
          f"global {res['g'][0]:.2f} ms ({upd / res['g'][0] / 1e9:.2f}e12/s), identical={same}")
    del idx, val, ws2
    torch.cuda.empty_cache()
