"""Run the factored Gram once on a config shape (for ncu)."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2505_21404_b200 as P  # noqa: E402
from paper_2505_21404_b200 import kernels as K  # noqa: E402

cfg = {"2": ("heat1d", (2, 64, 64, 64, 64, 1), (2000, 400, 400)),
       "3": ("poisson5d_sin", (5, 512, 512, 512, 512, 1), (3500, 500))}[sys.argv[1] if len(sys.argv) > 1 else "2"]
prob = P.make_problem(cfg[0])
spec = P.MlpSpec(cfg[1])
rmap = P.PinnResidualMap(prob, spec, prob.sample(cfg[2], np.random.default_rng(0)))
theta = P.xavier_normal_params(spec)
d = rmap._device()
r = torch.empty(rmap.m, dtype=torch.float64, device="cuda")
Kf = torch.empty(rmap.m, rmap.m, dtype=torch.float64, device="cuda")
ws = K.workspace("pinn", d["ws_bytes"])
for _ in range(2):
    K.gram_factored(d["mlp"], theta.tensor, d["arr"], d["nclass"], r, Kf, ws)
torch.cuda.synchronize()
print("ok", float(Kf.norm()))
