"""Jacobi eigensolver timing and sweep count on a config-5 landmark block (GPU)."""
import sys
import time

import numpy as np
import torch

sys.path.insert(0, ".")
import paper_2505_21404_b200 as P  # noqa: E402
from paper_2505_21404_b200 import kernels as K  # noqa: E402

prob = P.make_problem("poisson2d")
spec = P.MlpSpec((2, 256, 256, 256, 256, 1))
rmap = P.PinnResidualMap(prob, spec, prob.sample((30000, 2000), np.random.default_rng(0)))
rmap.gram_mode = "factored"
theta = P.xavier_normal_params(spec)
lm = np.sort(np.random.default_rng(1).choice(32000, 512, replace=False))
Kc = rmap.kcols_t(theta, lm)
KII = Kc.index_select(0, torch.as_tensor(lm, device="cuda")).contiguous()
for _ in range(2):
    w, V, sw = K.syev_jacobi(KII, 512)
torch.cuda.synchronize()
t = time.perf_counter()
for _ in range(3):
    w, V, sw = K.syev_jacobi(KII, 512)
torch.cuda.synchronize()
dt = (time.perf_counter() - t) / 3
A = KII.cpu().numpy()
ref = np.linalg.eigvalsh(0.5 * (A + A.T))
print(f"jacobi 512: {dt*1e3:.2f} ms, sweeps {int(sw.item())}, max|dev| / lmax "
      f"{np.abs(np.sort(w.cpu().numpy()) - np.sort(np.abs(ref))).max() / ref[-1]:.2e}, "
      f"kept {(w > 1e-10 * w.max()).sum().item()} vs ref {(ref > 1e-10 * ref[-1]).sum()}")
for _ in range(2):
    torch.linalg.eigh(KII)
torch.cuda.synchronize()
t = time.perf_counter()
for _ in range(3):
    torch.linalg.eigh(KII)
torch.cuda.synchronize()
print(f"torch.linalg.eigh 512: {(time.perf_counter() - t) / 3 * 1e3:.2f} ms")
