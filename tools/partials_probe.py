"""K-means partial sums alone (skc_kmeans_partials_csc through SketchKMeans.partials) at a BASELINE
K-means config: time per call. usage: python tools/partials_probe.py [c2|c5] [reps]"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

import bench
import paper_1511_00152_b200 as skc

wl = sys.argv[1] if len(sys.argv) > 1 else "c2"
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 30
cfg = bench.WORKLOADS[wl]
n = cfg["n"]
dev = torch.device("cuda", 0)
X = bench.gen_rows(wl, n, 0, dev, torch)
spec = skc.PreconditionSpec.create("hadamard", cfg["p"], sign_seed=bench.derive_seed(2026, 0xD5))
plan = skc.SamplingPlan(bench.derive_seed(2026, 0x5A), spec.p_pad, cfg["m"])
sk = skc.sketch_stream(skc.RowSource(X), spec, plan, compute="f64")
ops = skc.SketchKMeans(sk)
K = cfg["K"]
labels = torch.as_tensor(np.random.default_rng(1).integers(0, K, n).astype(np.int32), device=dev)
ops.partials(labels, K)
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(reps):
    r = ops.partials(labels, K)
e1.record()
torch.cuda.synchronize()
print(f"{wl} partials: {e0.elapsed_time(e1) / reps * 1e3:.1f} us per call; checksum {float(r[0].sum()):.12e} "
      f"env TILE_SMALL={os.environ.get('SKC_TILE_SMALL')} DBG={os.environ.get('SKC_TS_DBG')}")
