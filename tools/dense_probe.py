"""Second-pass kernels (K8 dense assign, K9 cluster sums) on HBM-resident rows: time and GB/s."""
import sys

import torch

sys.path.insert(0, __import__("os").path.dirname(__import__("os").path.dirname(__import__("os").path.abspath(__file__))))
from paper_1511_00152_b200 import _lib  # noqa: E402

dev = torch.device("cuda")
L = _lib.lib()
for n, p, K, dt in ((1 << 22, 1024, 10, torch.float32), (1 << 20, 2048, 100, torch.float32),
                    (1 << 22, 1024, 10, torch.float64)):
    X = torch.randn((n, p), device=dev, dtype=dt)
    mu = torch.randn((K, p), device=dev, dtype=torch.float64)
    lab = torch.randint(0, K, (n,), device=dev, dtype=torch.int32)
    lab2 = torch.empty(n, dtype=torch.int32, device=dev)
    d2 = torch.empty(n, dtype=torch.float64, device=dev)
    aws = _lib.workspace(L.skc_dense_assign_workspace(p, K), dev)
    sums = torch.zeros((K, p), dtype=torch.float64, device=dev)
    cnt = torch.zeros(K, dtype=torch.int64, device=dev)
    ws = _lib.workspace(L.skc_dense_sums_workspace(n, p, K), dev)
    st = _lib.stream_ptr(dev)
    xc = _lib.dtype_code(X)

    def a():
        _lib.call("skc_dense_assign", X.data_ptr(), xc, p, n, p, mu.data_ptr(), K, aws.data_ptr(), lab2.data_ptr(),
                  d2.data_ptr(), st)

    def s():
        _lib.call("skc_dense_sums", X.data_ptr(), xc, p, n, p, lab.data_ptr(), K, sums.data_ptr(), cnt.data_ptr(),
                  ws.data_ptr(), st)

    for name, f in (("assign", a), ("sums", s)):
        f()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(5):
            f()
        e1.record()
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1) / 5
        gb = n * p * X.element_size() / 1e9
        print(f"n={n} p={p} K={K} {str(dt)[6:]}: {name} {ms:.3f} ms -> {gb / (ms * 1e-3):.0f} GB/s of rows")
    del X
