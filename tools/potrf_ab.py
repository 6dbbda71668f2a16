"""potrf check + timing (DNGD_POTRF_DATAFLOW=1 selects the persistent dataflow schedule)."""
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2505_21404_b200 import kernels as Kn  # noqa: E402


def timed(fn, iters=10):
    fn()
    torch.cuda.synchronize()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    for _ in range(iters):
        fn()
    e.record()
    torch.cuda.synchronize()
    return s.elapsed_time(e) / iters


dev = torch.device("cuda")
torch.manual_seed(0)
path = "dataflow" if os.environ.get("DNGD_POTRF_DATAFLOW") else "panels"
for m in (1, 63, 64, 65, 130, 1020, 2800, 2803, 4000, 8000):
    A = torch.randn(m, m + 16, dtype=torch.float64, device=dev)
    Km = (A @ A.T) / m
    fac = Kn.CholeskyFactor(m, dev)
    fac.factor(Km, 1e-3)
    torch.cuda.synchronize()
    Lref = torch.linalg.cholesky(Km + 1e-3 * torch.eye(m, dtype=torch.float64, device=dev))
    L = torch.tril(fac.L[:m, :m])
    err = float((L - Lref).norm() / Lref.norm())
    b = torch.randn(m, dtype=torch.float64, device=dev)
    x = b.clone()
    fac.solve_(x)
    res = float(((Km + 1e-3 * torch.eye(m, dtype=torch.float64, device=dev)) @ x - b).norm() / b.norm())
    t = timed(lambda: fac.factor(Km, 1e-3))
    print(json.dumps({"path": path, "m": m, "ms": t, "rel_err_vs_cusolver": err, "solve_res": res,
                      "info": int(fac.info.item())}), flush=True)
# failing pivot: indefinite matrix, pivot 71 breaks
m = 300
Km = torch.eye(m, dtype=torch.float64, device=dev)
Km[70, 70] = -5.0
fac = Kn.CholeskyFactor(m, dev)
fac.factor(Km, 0.0)
torch.cuda.synchronize()
print(json.dumps({"path": path, "failing_info": int(fac.info.item()), "expect": 71}), flush=True)
