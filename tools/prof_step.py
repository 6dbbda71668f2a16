"""Run a few pieces once for ncu launch lists: potrf/potrs at m, or one bench step."""
import argparse, os, sys
import numpy as np, torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2505_21404_b200 import kernels as K

ap = argparse.ArgumentParser()
ap.add_argument("--what", default="potrf")
ap.add_argument("--m", type=int, default=2800)
a = ap.parse_args()
m = a.m
A = torch.randn(m, m + 16, dtype=torch.float64, device="cuda")
Km = (A @ A.T) / m
fac = K.CholeskyFactor(m, "cuda")
b = torch.randn(m, dtype=torch.float64, device="cuda")
for _ in range(2):
    fac.factor(Km, 1e-3)
    fac.solve_(b)
torch.cuda.synchronize()
print("info", int(fac.info.item()))
