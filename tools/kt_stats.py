"""Per-iteration candidate statistics of the K5t filter on a C5-shaped Lloyd run.
usage: python tools/kt_stats.py [iters] [n]"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import bench  # noqa: E402
import paper_1511_00152_b200 as skc  # noqa: E402
from paper_1511_00152_b200 import cluster  # noqa: E402

wl = "c5"
cfg = bench.WORKLOADS[wl]
iters = int(sys.argv[1]) if len(sys.argv) > 1 else cfg["iters"]
n = int(sys.argv[2]) if len(sys.argv) > 2 else cfg["n"]
dev = torch.device("cuda", 0)
X = bench.gen_rows(wl, n, 0, dev, torch)
spec = skc.PreconditionSpec.create("hadamard", cfg["p"], sign_seed=bench.derive_seed(2026, 0xD5))
plan = skc.SamplingPlan(bench.derive_seed(2026, 0x5A), spec.p_pad, cfg["m"])
sk = skc.sketch_stream(skc.RowSource(X), spec, plan, compute="f64")
del X
ops = skc.SketchKMeans(sk)
p, K = spec.p_pad, cfg["K"]
K4, Npad = (K + 3) & ~3, (K + 15) & ~15
r256 = lambda b: (b + 255) & ~255  # noqa: E731
off_ncand = r256(p * K * 16) + r256(p * K4 * 4) + r256((p // 32) * Npad * 64 * 2) + r256(n * 8)
orig = cluster.SketchKMeans.assign


def assign(self, mu, prev, labels, d2min, out, d2max):
    orig(self, mu, prev, labels, d2min, out, d2max)
    ws = self._ws.get(("assign_tc", mu.shape[1]))
    if ws is None or prev is None:
        return
    nc = ws[off_ncand:off_ncand + self.n].cpu().numpy()
    h = np.bincount(np.where(nc == 255, 9, nc), minlength=10)
    print("ncand histogram (0..8, overflow):", h.tolist(), flush=True)


cluster.SketchKMeans.assign = assign
mu = ops.init_centers(np.random.default_rng(2026).choice(n, K, replace=False))
lab, mu1, traj, it, secs = ops.lloyd(mu, iters)
print(f"{it} iterations")
