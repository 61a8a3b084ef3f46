"""Wall time of successive sparsified_kmeans calls from pinned host rows (C2 shape): where the
e2e line's run-to-run variance comes from."""
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
import paper_1511_00152_b200 as skc  # noqa: E402

wl = sys.argv[1] if len(sys.argv) > 1 else "c2"
cfg = bench.WORKLOADS[wl]
n, p, m, K = cfg["n"], cfg["p"], cfg["m"], cfg["K"]
dev = torch.device("cuda")
host = torch.empty((n, p), dtype=torch.float32, pin_memory=True)
host.copy_(bench.gen_rows(wl, n, 0, dev, torch).cpu())
chosen = np.random.default_rng(bench.SEED).choice(n, K, replace=False)
src = skc.RowSource(host, chunk_cols=1 << 16)
for it in range(6):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    r = skc.sparsified_kmeans(src, K, m / p, max_iter=cfg["iters"], seed=bench.SEED, init=chosen)
    t1 = time.perf_counter()
    print(f"call {it}: {1e3 * (t1 - t0):.2f} ms, iterations {r.diagnostics['iterations']}", flush=True)

import cProfile  # noqa: E402
import pstats  # noqa: E402

pr = cProfile.Profile()
pr.enable()
for it in range(6):
    skc.sparsified_kmeans(src, K, m / p, max_iter=cfg["iters"], seed=bench.SEED, init=chosen)
torch.cuda.synchronize()
pr.disable()
pstats.Stats(pr).sort_stats("cumulative").print_stats(25)
