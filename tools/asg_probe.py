"""K-means assignment kernel alone (skc_kmeans_assign) on a synthetic sketch: time + checksum.
usage: python tools/asg_probe.py p m K n reps"""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1511_00152_b200 import _lib  # noqa: E402

dev = torch.device("cuda")
p, m, K, n, reps = (int(x) for x in (sys.argv[1:6] if len(sys.argv) > 5 else (512, 26, 10, 200000, 20)))
L = _lib.lib()
st = _lib.stream_ptr(dev)
idx = torch.empty((n, m), dtype=torch.int32, device=dev)
_lib.call("skc_indices_philox", 7, 0, n, p, m, idx.data_ptr(), st)
g = torch.Generator(device=dev).manual_seed(5)
val = torch.randn((n, m), device=dev, generator=g, dtype=torch.float64)
mu = torch.randn((p, K), device=dev, generator=g, dtype=torch.float64) * 0.3
labels = torch.empty(n, dtype=torch.int32, device=dev)
prev = torch.zeros(n, dtype=torch.int32, device=dev)
d2 = torch.empty(n, dtype=torch.float64, device=dev)
out = torch.zeros(2, dtype=torch.int64, device=dev)
d2max = torch.zeros(1, dtype=torch.float64, device=dev)
ws = _lib.workspace(L.skc_kmeans_assign_workspace(n, p, K), dev)


def run():
    _lib.call("skc_kmeans_assign", idx.data_ptr(), val.data_ptr(), _lib.F64, n, m, mu.data_ptr(), p, K, prev.data_ptr(),
              labels.data_ptr(), d2.data_ptr(), out.data_ptr(), d2max.data_ptr(), ws.data_ptr(), ws.numel(), st)


run()
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(reps):
    run()
e1.record()
torch.cuda.synchronize()
t = e0.elapsed_time(e1) / reps
cs = int((labels.to(torch.int64) * torch.arange(n, device=dev)).sum().item())
print(f"assign p={p} m={m} K={K} n={n}: {t * 1e3:.1f} us  labels-checksum {cs} d2sum {float(d2.sum()):.12e} changed {int(out[0])}")
