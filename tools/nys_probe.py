"""Timing and rank of the Nystrom build pieces at config 5 (GPU)."""
import sys
import time

import numpy as np
import torch

sys.path.insert(0, ".")
import paper_2505_21404_b200 as P  # noqa: E402
from paper_2505_21404_b200 import kernels as K  # noqa: E402
from paper_2505_21404_b200 import solver as S  # noqa: E402

prob = P.make_problem("poisson2d")
spec = P.MlpSpec((2, 256, 256, 256, 256, 1))
rmap = P.PinnResidualMap(prob, spec, prob.sample((30000, 2000), np.random.default_rng(0)))
rmap.gram_mode = "factored"
theta = P.xavier_normal_params(spec)
lm = np.sort(np.random.default_rng(1).choice(32000, 512, replace=False))
Kc = rmap.kcols_t(theta, lm)
KII = Kc.index_select(0, torch.as_tensor(lm, device="cuda")).contiguous()
Lt = torch.zeros((512, 512), dtype=torch.float64, device="cuda")
kd = torch.zeros(1, dtype=torch.int32, device="cuda")


def timed(fn, reps=3):
    fn()
    torch.cuda.synchronize()
    t = time.perf_counter()
    for _ in range(reps):
        out = fn()
    torch.cuda.synchronize()
    return (time.perf_counter() - t) / reps * 1e3, out


t_pc, _ = timed(lambda: K.pivoted_cholesky(KII, 512, S.PIVCHOL_TOL, Lt, kd))
k = int(kd.item())
G0 = K.gemm_nt(Lt[:k], Lt[:k], K=512)
t_j, out = timed(lambda: K.syev_jacobi(G0, k))
t_all, _ = timed(lambda: S.nystrom_from_columns(Kc, lm, 1e-5))
print(f"k = {k}; pivchol {t_pc:.2f} ms, jacobi(k) {t_j:.2f} ms ({int(out[2].item())} sweeps), "
      f"nystrom_from_columns {t_all:.2f} ms")
