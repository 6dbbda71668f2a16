"""One emulated-FP64 factored Gram launch at BASELINE config 3 (for ncu)."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2505_21404_b200 as P  # noqa: E402
from paper_2505_21404_b200 import kernels as K  # noqa: E402

S = int(sys.argv[1]) if len(sys.argv) > 1 else 7
prob = P.make_problem("poisson5d_sin")
spec = P.MlpSpec((5, 512, 512, 512, 512, 1))
rmap = P.PinnResidualMap(prob, spec, prob.sample((3500, 500), np.random.default_rng(0)))
theta = P.xavier_normal_params(spec)
d = rmap._device()
rmap.residuals_act_t(theta)
ws = rmap._act_workspace()
Kt = torch.zeros(rmap.m, rmap.m, dtype=torch.float64, device="cuda")
for _ in range(2):
    K.gram_factored_act(d["mlp"], d["arr"], d["nclass"], Kt, ws, slices=S)
torch.cuda.synchronize()
print("ok")
