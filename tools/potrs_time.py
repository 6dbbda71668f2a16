"""potrs (forward + backward block substitution) timing and backward error vs m."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2505_21404_b200 import kernels as Kn  # noqa: E402

dev = torch.device("cuda")
for m in [int(x) for x in sys.argv[1:]] or [1020, 2800, 4000, 8000]:
    A = torch.randn(m, m, dtype=torch.float64, device=dev)
    Km = A @ A.T / m + 1e-3 * torch.eye(m, dtype=torch.float64, device=dev)
    fac = Kn.CholeskyFactor(m, dev)
    fac.factor(Km, 0.0)
    b = torch.randn(m, dtype=torch.float64, device=dev)
    x = b.clone()
    for _ in range(3):
        x.copy_(b)
        fac.solve_(x)
    torch.cuda.synchronize()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    for _ in range(20):
        fac.solve_(x)
    e.record()
    torch.cuda.synchronize()
    x.copy_(b)
    fac.solve_(x)
    berr = float(torch.linalg.norm(Km @ x - b) / (torch.linalg.matrix_norm(Km, 2) * torch.linalg.norm(x) + torch.linalg.norm(b)))
    print(f"m={m}: potrs {s.elapsed_time(e) / 20 * 1e3:.1f} us, backward error {berr:.2e}", flush=True)
