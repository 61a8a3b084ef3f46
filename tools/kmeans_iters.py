"""One C2/C5 Lloyd run of `iters` iterations (for per-launch ncu timing in order).
usage: python tools/kmeans_iters.py c5 [iters] [n]"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import bench  # noqa: E402
import paper_1511_00152_b200 as skc  # noqa: E402

wl = sys.argv[1] if len(sys.argv) > 1 else "c5"
cfg = bench.WORKLOADS[wl]
iters = int(sys.argv[2]) if len(sys.argv) > 2 else cfg["iters"]
n = int(sys.argv[3]) if len(sys.argv) > 3 else cfg["n"]
dev = torch.device("cuda", 0)
X = bench.gen_rows(wl, n, 0, dev, torch)
spec = skc.PreconditionSpec.create("hadamard", cfg["p"], sign_seed=bench.derive_seed(2026, 0xD5))
plan = skc.SamplingPlan(bench.derive_seed(2026, 0x5A), spec.p_pad, cfg["m"])
sk = skc.sketch_stream(skc.RowSource(X), spec, plan, compute="f64")
del X
ops = skc.SketchKMeans(sk)
mu = ops.init_centers(np.random.default_rng(2026).choice(n, cfg["K"], replace=False))
lab, mu1, traj, it, secs = ops.lloyd(mu, iters)
torch.cuda.synchronize()
print(f"{wl}: {it} iterations, {secs * 1e3:.1f} ms, objective {traj[-1]:.6e}")
