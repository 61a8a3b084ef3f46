"""K3t probe: accuracy against the accumulation window, and tc vs scatter time across m/p.

usage (GPU box): python tools/covtc_probe.py [acc|time|all]
"""
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1511_00152_b200 as skc  # noqa: E402
from oracle import oracle as O  # noqa: E402


def rel_fro(a, b):
    return float(np.linalg.norm(a - b) / np.linalg.norm(b))


def accuracy():
    for p, m, n in [(256, 64, 5000), (1024, 51, 30000), (1024, 256, 20000)]:
        rng = np.random.default_rng(p + m)
        X = (rng.standard_t(3, size=(p, n)) / np.sqrt(3.0)).astype(np.float32)
        spec = skc.PreconditionSpec.create("hadamard", p, 3)
        sk = skc.sketch_stream(X, spec, skc.SamplingPlan(4, p, m), compute="f32")
        Co = O.estimate_covariance(sk.host_indices(), sk.host_values().astype(np.float64), p, nthreads=8)
        os.environ["SKC_COV_PATH"] = "tc"
        errs = []
        for w in (1, 4, 8, 16, 32, 64):
            os.environ["SKC_COVTC_WINDOW"] = str(w)
            C = skc.estimate_covariance(sk).matrix
            d = np.diag(C) / np.diag(Co) - 1
            errs.append(f"w={w}: fro {rel_fro(C, Co):.2e} diag mean {d.mean():+.2e}")
        os.environ.pop("SKC_COVTC_WINDOW")
        os.environ["SKC_COV_PATH"] = "band"
        try:
            eb = rel_fro(skc.estimate_covariance(sk).matrix, Co)
        except Exception as e:  # noqa: BLE001
            eb = str(e)[:40]
        print(f"p={p} m={m} n={n}: band {eb}; tc " + "; ".join(errs), flush=True)


def timing():
    L = skc._lib
    lib = L.lib()
    dev = torch.device("cuda")
    p = int(os.environ.get("PROBE_P", "1024"))
    n = int(os.environ.get("PROBE_N", str(1 << 22)))
    ms_list = [int(x) for x in os.environ.get("PROBE_M", "32,51,64,96,128,192,256").split(",")]
    for m in ms_list:
        g = torch.Generator(device=dev).manual_seed(m)
        idx = torch.empty((n, m), dtype=torch.int32, device=dev)  # sorted uniform m-subsets
        L.call("skc_indices_philox", m + 7, 0, n, p, m, idx.data_ptr(), L.stream_ptr(dev))
        val = torch.randn((n, m), device=dev, generator=g, dtype=torch.float32)
        stats = torch.zeros(3, dtype=torch.float64, device=dev)
        acc = torch.zeros(p, dtype=torch.float64, device=dev)
        wsm = L.workspace(lib.skc_moments_workspace(n, m, p), dev)
        L.call("skc_moments", idx.data_ptr(), val.data_ptr(), L.F32, n, m, p, acc.data_ptr(), stats.data_ptr(),
               wsm.data_ptr(), wsm.numel(), L.stream_ptr(dev))
        tri = torch.zeros(p * (p + 1) // 2, dtype=torch.float64, device=dev)
        row = [f"m={m:4d} (m/p={m / p:.3f})"]
        for path in os.environ.get("PROBE_PATHS", "band,tc").split(","):
            os.environ["SKC_COV_PATH"] = path
            try:
                ws = L.workspace(lib.skc_cov_workspace(n, m, p), dev)
                f = lambda: L.call("skc_cov_accumulate", idx.data_ptr(), val.data_ptr(), L.F32, n, m, p,  # noqa
                                   stats.data_ptr(), tri.data_ptr(), ws.data_ptr(), ws.numel(), L.stream_ptr(dev))
                f()
                torch.cuda.synchronize()
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                e0.record()
                for _ in range(3):
                    f()
                e1.record()
                torch.cuda.synchronize()
                ms = e0.elapsed_time(e1) / 3
                row.append(f"{path} {ms:7.2f} ms ({n * 1e-6 / ms:6.1f} G samples/s)")
            except Exception as e:  # noqa: BLE001
                row.append(f"{path} n/a ({str(e)[:30]})")
            del ws
        os.environ.pop("SKC_COV_PATH")
        print("  ".join(row), flush=True)
        del idx, val


if __name__ == "__main__":
    what = sys.argv[1] if len(sys.argv) > 1 else "all"
    t = time.time()
    if what in ("acc", "all"):
        accuracy()
    if what in ("time", "all"):
        timing()
    print(f"done in {time.time() - t:.1f} s")
