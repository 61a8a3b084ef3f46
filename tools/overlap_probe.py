"""Can the ALU-bound oracle index kernel and the HBM-bound gather kernel overlap?

Times K1a (skc_indices) alone, K1b (skc_sketch_given) alone, and both launched at once on two
streams over independent buffers, for index-kernel occupancy caps (SKC_IDX_OCC).
usage (GPU box): python tools/overlap_probe.py
"""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1511_00152_b200 as skc  # noqa: E402

L = skc._lib
dev = torch.device("cuda")
n, p, m = 1 << 24, 1024, 51
X = torch.randn((n, p), device=dev, dtype=torch.float32)
idx = torch.empty((n, m), dtype=torch.int32, device=dev)
idx2 = torch.empty_like(idx)
val = torch.empty((n, m), dtype=torch.float32, device=dev)
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
L.call("skc_indices", 7, 0, n, p, m, idx.data_ptr(), L.stream_ptr(dev))
torch.cuda.synchronize()


def ind(s, rows=n):
    L.call("skc_indices", 7, 0, rows, p, m, idx2.data_ptr(), s.cuda_stream)


def gat(s, rows=n):
    L.call("skc_sketch_given", X.data_ptr(), L.F32, p, rows, p, p, 0, 11, m, L.F32, idx.data_ptr(), val.data_ptr(),
           L.F32, s.cuda_stream)


def timed(fn, reps=3):
    fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        fn()
    # join both streams into the current one
    ev = torch.cuda.Event()
    for s in (s1, s2):
        ev.record(s)
        torch.cuda.current_stream().wait_event(ev)
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps


def both():
    cur = torch.cuda.current_stream()
    for s in (s1, s2):
        s.wait_stream(cur)
    ind(s1)
    gat(s2)


for gocc, iocc in (("3", "8"), ("2", "3"), ("2", "4"), ("1", "5"), ("1", "6"), ("2", "2")):
    os.environ["SKC_IDX_OCC"] = iocc
    os.environ["SKC_GATHER_OCC"] = gocc
    a = timed(lambda: ind(torch.cuda.current_stream()))
    b = timed(lambda: gat(torch.cuda.current_stream()))
    c = timed(both)
    print(f"gather occ {gocc} idx occ {iocc}: indices {a:6.2f} ms, gather {b:6.2f} ms, sum {a + b:6.2f}, "
          f"concurrent {c:6.2f} ms", flush=True)
