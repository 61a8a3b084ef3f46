"""Host (LAPACK via numpy) vs device (cuSOLVER syevd) top-k eigensolve times at the C3/C4 sizes."""
import sys
import time

import numpy as np
import torch

sys.path.insert(0, __import__("os").path.dirname(__import__("os").path.dirname(__import__("os").path.abspath(__file__))))
from paper_1511_00152_b200.estimators import top_eigenvectors  # noqa: E402

for p in (1024, 4096):
    rng = np.random.default_rng(p)
    A = rng.standard_normal((p, p))
    C = A @ A.T / p
    Cd = torch.as_tensor(C, device="cuda")
    top_eigenvectors(Cd, 10, solver="device")
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    Vd = top_eigenvectors(Cd, 10, solver="device")
    torch.cuda.synchronize()
    td = time.perf_counter() - t0
    t0 = time.perf_counter()
    Vh = top_eigenvectors(C, 10)
    th = time.perf_counter() - t0
    err = np.abs(np.abs(Vd.cpu().numpy().T @ Vh) - np.eye(10)).max()
    print(f"p={p}: host eigh {th * 1e3:.1f} ms, device eigh {td * 1e3:.1f} ms, |V_d^T V_h| - I max {err:.2e}")
