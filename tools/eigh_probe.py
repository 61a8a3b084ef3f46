"""Host LAPACK eigh vs the device top-k solver (skc_top_eigenvectors: cuSOLVER syevdx over an
index range) vs the full device syevd (torch.linalg.eigh) at the C3/C4 sizes, k = 20."""
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1511_00152_b200.estimators import top_eigenvectors  # noqa: E402


def timed(f, reps=3):
    f()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(reps):
        r = f()
    torch.cuda.synchronize()
    return r, (time.perf_counter() - t0) / reps


for p in (1024, 4096):
    k = 20
    rng = np.random.default_rng(p)
    A = rng.standard_normal((p, p))
    C = A @ A.T / p + np.diag(np.linspace(30.0, 10.0, p) * (np.arange(p) < k))  # k separated spikes
    Cd = torch.as_tensor(C, device="cuda")
    Vd, td = timed(lambda: top_eigenvectors(Cd, k, solver="device"))
    _, tf = timed(lambda: torch.linalg.eigh(0.5 * (Cd + Cd.T))[1].flip(1)[:, :k].contiguous())
    t0 = time.perf_counter()
    Vh = top_eigenvectors(C, k)
    th = time.perf_counter() - t0
    err = np.abs(np.abs(Vd.cpu().numpy().T @ Vh) - np.eye(k)).max()
    print(f"p={p} k={k}: host eigh {th * 1e3:.1f} ms, device top-k syevdx {td * 1e3:.1f} ms, "
          f"device full syevd {tf * 1e3:.1f} ms, max ||V_d^T V_h| - I| {err:.2e}")
