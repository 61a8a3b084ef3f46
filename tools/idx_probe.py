"""Oracle-mode index kernel alone (skc_indices) at a given (p, m, n): time and sanity."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1511_00152_b200 import _lib  # noqa: E402

dev = torch.device("cuda")
p = int(sys.argv[1]) if len(sys.argv) > 1 else 1024
m = int(sys.argv[2]) if len(sys.argv) > 2 else 51
n = int(sys.argv[3]) if len(sys.argv) > 3 else 1 << 24
reps = int(sys.argv[4]) if len(sys.argv) > 4 else 3
idx = torch.empty((n, m), dtype=torch.int32, device=dev)
st = _lib.stream_ptr(dev)
run = lambda: _lib.call("skc_indices", 0x1234, 0, n, p, m, idx.data_ptr(), st)  # noqa: E731
run()
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(reps):
    run()
e1.record()
torch.cuda.synchronize()
t = e0.elapsed_time(e1) / reps
h = int(torch.sum(idx[:: max(1, n // 4096)].to(torch.int64) * 2654435761 % 1000003).item())
print(f"indices p={p} m={m} n={n}: {t:.3f} ms ({n / t / 1e6:.1f} M rows/s) checksum {h}")
