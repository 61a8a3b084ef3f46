"""Time the pieces of one sparsified Lloyd iteration at a BASELINE K-means config."""
import sys, time, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import bench
import paper_1511_00152_b200 as skc

wl = sys.argv[1] if len(sys.argv) > 1 else "c2"
n = int(sys.argv[2]) if len(sys.argv) > 2 else bench.WORKLOADS[wl]["n"]
cfg = bench.WORKLOADS[wl]
dev = torch.device("cuda", 0)
X = bench.gen_rows(wl, n, 0, dev, torch)
spec = skc.PreconditionSpec.create("hadamard", cfg["p"], sign_seed=bench.derive_seed(2026, 0xD5))
plan = skc.SamplingPlan(bench.derive_seed(2026, 0x5A), spec.p_pad, cfg["m"])
for vt in ("f64", "f32"):
    sk = skc.sketch_stream(skc.RowSource(X), spec, plan, compute=vt)
    ops = skc.SketchKMeans(sk)
    mu = ops.init_centers(np.random.default_rng(2026).choice(n, cfg["K"], replace=False))
    lab = torch.empty(n, dtype=torch.int32, device=dev); d2 = torch.empty(n, dtype=torch.float64, device=dev)
    out = torch.zeros(2, dtype=torch.int64, device=dev); mx = torch.zeros(1, dtype=torch.float64, device=dev)
    obj = torch.zeros(1, dtype=torch.float64, device=dev)
    def t(fn, reps=20):
        fn(); torch.cuda.synchronize()
        e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(reps): fn()
        e1.record(); e1.synchronize(); return e0.elapsed_time(e1) / reps
    ta = t(lambda: ops.assign(mu, None, lab, d2, out, mx))
    tp = t(lambda: ops.objective(d2, obj))
    tu = t(lambda: ops.update(lab, mu))
    tl = t(lambda: ops.lloyd(mu, cfg["iters"]), 3)
    _, _, _, its, _ = ops.lloyd(mu, cfg["iters"])
    print(f"{wl} n={n} values={vt}: assign {ta:.3f} ms, pairwise {tp:.3f} ms, update {tu:.3f} ms, "
          f"lloyd({its} it) {tl:.3f} ms -> {n*its/(tl*1e-3):.3e} point-iters/s")
