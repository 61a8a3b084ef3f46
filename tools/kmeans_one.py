import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch, bench
import paper_1511_00152_b200 as skc
wl = sys.argv[1] if len(sys.argv) > 1 else "c2"
cfg = bench.WORKLOADS[wl]; n = int(sys.argv[2]) if len(sys.argv) > 2 else cfg["n"]
dev = torch.device("cuda", 0)
X = bench.gen_rows(wl, n, 0, dev, torch)
spec = skc.PreconditionSpec.create("hadamard", cfg["p"], sign_seed=bench.derive_seed(2026, 0xD5))
plan = skc.SamplingPlan(bench.derive_seed(2026, 0x5A), spec.p_pad, cfg["m"])
sk = skc.sketch_stream(skc.RowSource(X), spec, plan, compute="f64")
ops = skc.SketchKMeans(sk)
mu = ops.init_centers(np.random.default_rng(2026).choice(n, cfg["K"], replace=False))
ops.lloyd(mu, 2); torch.cuda.synchronize()
ops.lloyd(mu, 2); torch.cuda.synchronize()
