"""potrf vs cuSOLVER over a size sweep (well-conditioned SPD: A A^T / m + I)."""
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2505_21404_b200 import kernels as Kn  # noqa: E402

dev = torch.device("cuda")
torch.manual_seed(0)
sizes = [int(x) for x in sys.argv[1:]] or [4032, 4096, 4160, 4500, 5000, 6000, 7000, 8000]
for m in sizes:
    A = torch.randn(m, m, dtype=torch.float64, device=dev)
    Km = (A @ A.T) / m + torch.eye(m, dtype=torch.float64, device=dev)
    fac = Kn.CholeskyFactor(m, dev)
    fac.factor(Km, 0.0)
    torch.cuda.synchronize()
    Lref = torch.linalg.cholesky(Km)
    L = torch.tril(fac.L[:m, :m])
    d = (L - Lref).abs()
    bad = (d > 1e-10 * Lref.abs().max()).nonzero()
    first = bad[0].tolist() if len(bad) else None
    print(json.dumps({"m": m, "rel_err": float((L - Lref).norm() / Lref.norm()), "first_bad": first,
                      "nbad": int(len(bad)), "info": int(fac.info.item())}), flush=True)
