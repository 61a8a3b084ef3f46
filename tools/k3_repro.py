"""C3-shape covariance on the bench generator (one chunk), for sanitizer runs of K3."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
import paper_1511_00152_b200 as skc  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 1 << 16
comp = sys.argv[2] if len(sys.argv) > 2 else "f64"
c = bench.CONFIGS["c3"] if hasattr(bench, "CONFIGS") else None
p, m = 1024, 51
X = bench.gen_rows("c3", n, 0, torch.device("cuda"), torch)
spec = skc.PreconditionSpec.create("hadamard", p, 11)
plan = skc.SamplingPlan(12, p, m)
mom = skc.stream_moments(skc.RowSource(X), spec, plan, compute=comp)
C = skc.covariance_from_moments(mom, p, m, n).cpu()
torch.cuda.synchronize()
print("ok", float(C.abs().max()))
