"""Kernel timeline of one potrf (torch.profiler / CUPTI): start, duration, stream."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2505_21404_b200 import kernels as Kn  # noqa: E402

m = int(sys.argv[1]) if len(sys.argv) > 1 else 2800
torch.manual_seed(0)
A = torch.randn(m, m + 16, dtype=torch.float64, device="cuda")
Km = (A @ A.T) / m
fac = Kn.CholeskyFactor(m, "cuda")
for _ in range(3):
    fac.factor(Km, 1e-3)
torch.cuda.synchronize()
from torch.profiler import ProfilerActivity, profile  # noqa: E402

with profile(activities=[ProfilerActivity.CUDA]) as prof:
    fac.factor(Km, 1e-3)
    torch.cuda.synchronize()
evs = sorted((e for e in prof.events() if e.device_type.name == "CUDA"), key=lambda e: e.time_range.start)
t0 = evs[0].time_range.start
for e in evs[:60]:
    print(f"{e.time_range.start - t0:9.1f} {e.time_range.end - e.time_range.start:7.1f}  "
          f"{e.name[:60]}")
print("total", evs[-1].time_range.end - t0)
