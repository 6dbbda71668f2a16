"""A small dense D-NGD step (assembly, factored + materialised Gram, potrf, both
potrs, J^T w, f_vv, line search) and a small PCG step, for compute-sanitizer runs
(racecheck / memcheck / synccheck, one tool per run)."""
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
import paper_2505_21404_b200 as P  # noqa: E402

torch.cuda.set_device(0)
for pname, counts, widths, mode in [("heat1d", (150, 40, 40), (2, 32, 32, 1), "factored"),
                                    ("poisson2d", (200, 60), (2, 24, 24, 1), "materialized")]:
    prob = P.make_problem(pname)
    spec = P.MlpSpec(widths)
    rmap = P.PinnResidualMap(prob, spec, prob.sample(counts, np.random.default_rng(0)))
    rmap.gram_mode = mode
    theta = P.xavier_normal_params(spec)
    _, g = rmap.residuals_and_gradient(theta)
    res = P.dense_dual_solve(rmap, theta, g, lam=1e-3, use_ga=True)
    ls = P.device_line_search(rmap, theta, res.delta.tensor, rmap.loss(theta))
    pcg = P.pcg_step(rmap, theta, g, lam=1e-3, landmark_count=24, tol=1e-10, max_iters=50,
                     rng=np.random.default_rng(1))
torch.cuda.synchronize()
print("sanitize case ok", ls.eta, pcg.cg_iterations)
