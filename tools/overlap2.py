"""Round-2 overlap check: the oracle index kernel (occupancy-capped) beside the f64 TMA gather on a
second stream, full C3 size, independent buffers. usage: python tools/overlap2.py [idx_occ...]"""
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
val = torch.empty((n, m), dtype=torch.float64, device=dev)
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
L.call("skc_indices", 7, 0, n, p, m, idx.data_ptr(), L.stream_ptr(dev))
torch.cuda.synchronize()


def ind(s):
    L.call("skc_indices", 7, 0, n, p, m, idx2.data_ptr(), s.cuda_stream)


def gat(s):
    L.call("skc_sketch_given", X.data_ptr(), L.F32, p, n, p, p, 0, 11, m, L.F64, idx.data_ptr(), val.data_ptr(),
           L.F64, s.cuda_stream)


def timed(fn, reps=3):
    fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        fn()
    ev = torch.cuda.Event()
    for s in (s1, s2):
        ev.record(s)
        torch.cuda.current_stream().wait_event(ev)
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps


def both(first_gather):
    cur = torch.cuda.current_stream()
    for s in (s1, s2):
        s.wait_stream(cur)
    if first_gather:
        gat(s2)
        ind(s1)
    else:
        ind(s1)
        gat(s2)


for occ in sys.argv[1:] or ["2", "3", "4"]:
    os.environ["SKC_IDX_OCC"] = occ
    a = timed(lambda: ind(torch.cuda.current_stream()))
    b = timed(lambda: gat(torch.cuda.current_stream()))
    c = timed(lambda: both(True))
    d = timed(lambda: both(False))
    print(f"idx occ {occ}: indices {a:6.2f} ms, gather {b:6.2f} ms, sum {a + b:6.2f}, "
          f"concurrent gather-first {c:6.2f} ms, index-first {d:6.2f} ms", flush=True)
