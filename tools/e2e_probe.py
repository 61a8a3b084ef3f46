"""e2e anatomy at C3 shape: pure pinned H2D of the rows vs stream_moments vs sketch + moments."""
import sys
import time

import torch

sys.path.insert(0, __import__("os").path.dirname(__import__("os").path.dirname(__import__("os").path.abspath(__file__))))
import paper_1511_00152_b200 as skc  # noqa: E402
from paper_1511_00152_b200.sketch import device_row_chunks  # noqa: E402

dev = torch.device("cuda")
n, p, m = 1 << 21, 1024, 51
host = torch.randn((n, p), dtype=torch.float32).pin_memory()
spec = skc.PreconditionSpec.create("hadamard", p, 3)
plan = skc.SamplingPlan(5, p, m)


def timed(fn, reps=3):
    fn()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(reps):
        fn()
    torch.cuda.synchronize()
    return (time.perf_counter() - t0) / reps * 1e3


for chunk in (1 << 17, 1 << 15, 1 << 13):
    src = skc.RowSource(host, chunk_cols=chunk)

    def copy_only():
        for rows in device_row_chunks(src.row_chunks(), dev):
            pass

    def streamed():
        mom = skc.stream_moments(src, spec, plan, compute="f32")
        skc.covariance_from_moments(mom, p, m, n).cpu()

    def two_step():
        sk = skc.sketch_stream(src, spec, plan, compute="f32")
        mom = skc.accumulate_moments(sk)
        skc.covariance_from_moments(mom, p, m, n).cpu()

    tc, ts, tt = timed(copy_only), timed(streamed), timed(two_step)
    gb = n * p * 4 / 1e9
    print(f"chunk {chunk}: copy only {tc:.1f} ms ({gb / tc * 1e3:.1f} GB/s), stream_moments {ts:.1f} ms "
          f"({n / ts / 1e3:.2f} M/s), sketch+moments {tt:.1f} ms ({n / tt / 1e3:.2f} M/s)")
