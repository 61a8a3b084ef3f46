"""K3t operand limbs: accuracy of hi*hi only (fp16 products) against the banded scatter on C3 data,
for several accumulation windows. usage (GPU box): python tools/covtc_limbs.py [n]"""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
import paper_1511_00152_b200 as skc  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 1 << 22
for wl in ("c3", "c1big", "c4"):
    cfg = bench.WORKLOADS[wl]
    nn = min(n, 1 << 21) if wl == "c4" else n
    X = bench.gen_rows(wl, nn, 0, torch.device("cuda"), torch)
    spec = skc.PreconditionSpec.create("hadamard", cfg["p"], sign_seed=bench.derive_seed(2026, 0xD5))
    plan = skc.SamplingPlan(bench.derive_seed(2026, 0x5A), spec.p_pad, cfg["m"])
    sk = skc.sketch_stream(skc.RowSource(X), spec, plan, compute="f32")
    del X
    os.environ["SKC_COV_PATH"] = "g" if wl == "c4" else "b"
    Cb = skc.estimate_covariance(sk).matrix
    Cb = Cb.cpu().numpy() if hasattr(Cb, "cpu") else Cb
    for limbs in ("3", "1"):
        for w in ("8", "32"):
            os.environ.update(SKC_COV_PATH="t", SKC_COVTC_LIMBS=limbs, SKC_COVTC_WINDOW=w)
            C = skc.estimate_covariance(sk).matrix
            C = C.cpu().numpy() if hasattr(C, "cpu") else C
            e = np.linalg.norm(C - Cb) / np.linalg.norm(Cb)
            d = (np.diag(C) / np.diag(Cb) - 1).mean()
            print(f"{wl} n={nn} limbs={limbs} window={w}: rel fro {e:.2e}, diag mean {d:+.2e}", flush=True)
    for k in ("SKC_COV_PATH", "SKC_COVTC_LIMBS", "SKC_COVTC_WINDOW"):
        os.environ.pop(k, None)
