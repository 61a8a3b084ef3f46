import os, sys
sys.path.insert(0, os.getcwd())
import torch
import paper_1511_00152_b200 as skc
L = skc._lib; lib = L.lib(); dev = torch.device("cuda")
p, n, m = 1024, 1 << 20, int(os.environ.get("PM", "64"))
idx = torch.empty((n, m), dtype=torch.int32, device=dev)
L.call("skc_indices_philox", 5, 0, n, p, m, idx.data_ptr(), L.stream_ptr(dev))
val = torch.randn((n, m), device=dev, dtype=torch.float32)
stats = torch.tensor([float(n * m), 5.0, float(n)], dtype=torch.float64, device=dev)
tri = torch.zeros(p * (p + 1) // 2, dtype=torch.float64, device=dev)
os.environ["SKC_COV_PATH"] = "tc"
ws = L.workspace(lib.skc_cov_workspace(n, m, p), dev)
for _ in range(2):
    L.call("skc_cov_accumulate", idx.data_ptr(), val.data_ptr(), L.F32, n, m, p, stats.data_ptr(), tri.data_ptr(), ws.data_ptr(), ws.numel(), L.stream_ptr(dev))
torch.cuda.synchronize(); print("ok")
