"""The Nystrom eigen stage at config 5, piece by piece: pivoted Cholesky of K_II
(one CTA), L^T L, Jacobi on k x k -- CUDA-event times and the numerical rank k."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2505_21404_b200 as P  # noqa: E402
from paper_2505_21404_b200 import kernels as K  # noqa: E402
from paper_2505_21404_b200.solver import PIVCHOL_TOL  # noqa: E402

prob = P.make_problem("poisson2d")
spec = P.MlpSpec((2, 256, 256, 256, 256, 1))
rmap = P.PinnResidualMap(prob, spec, prob.sample((30000, 2000), np.random.default_rng(0)))
theta = P.xavier_normal_params(spec)
ell = 512
lm = np.sort(np.random.default_rng(1).choice(32000, ell, replace=False))
Kc = rmap.kcols_t(theta, lm)
KII = Kc.index_select(0, torch.as_tensor(lm, device="cuda")).contiguous()
Lt = torch.zeros((ell, ell), dtype=torch.float64, device="cuda")
kdev = torch.zeros(1, dtype=torch.int32, device="cuda")


def ev(fn, reps=5):
    fn()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(reps):
        fn()
    b.record()
    torch.cuda.synchronize()
    return a.elapsed_time(b) / reps


t_pc = ev(lambda: K.pivoted_cholesky(KII, ell, PIVCHOL_TOL, Lt, kdev))
k = int(kdev.item())
G0 = K.gemm_nt(Lt[:k], Lt[:k], K=ell)
t_g = ev(lambda: K.gemm_nt(Lt[:k], Lt[:k], K=ell))
t_j = ev(lambda: K.syev_jacobi(G0, k), reps=3)
_, _, sw = K.syev_jacobi(G0, k)
print(f"k = {k}: pivoted Cholesky {t_pc:.3f} ms, L^T L {t_g:.3f} ms, Jacobi {t_j:.3f} ms "
      f"({int(sw.item())} sweeps)")
