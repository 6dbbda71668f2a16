"""Sensitivity of the Nystrom preconditioner to the pivoted-Cholesky stop (GPU)."""
import sys

import numpy as np

sys.path.insert(0, ".")
import paper_2505_21404_b200 as P  # noqa: E402
from paper_2505_21404_b200 import solver as S  # noqa: E402

for pname, widths, counts in [("poisson2d", (2, 16, 16, 1), (90, 30)), ("heat1d", (2, 16, 16, 1), (60, 20, 20))]:
    problem = P.make_problem(pname)
    spec = P.MlpSpec(widths)
    colloc = problem.sample(counts, np.random.default_rng(21))
    theta = P.xavier_normal_params(spec)
    for tol in (1e-15, 1e-16, 1e-17, 0.0):
        S.PIVCHOL_TOL = tol
        out = {}
        for mode in ("factored", "materialized"):
            rmap = P.PinnResidualMap(problem, spec, colloc)
            rmap.gram_mode = mode
            pre = P.nystrom_build(rmap, theta, landmark_count=32, lam=1e-3, rng=np.random.default_rng(5))
            probe = np.random.default_rng(3).normal(size=rmap.m)
            out[mode] = (pre.apply(probe), pre.rank)
        a, b = out["factored"][0], out["materialized"][0]
        print(pname, tol, "rank", out["factored"][1], out["materialized"][1],
              "P^-1 rel diff %.2e" % (np.linalg.norm(a - b) / np.linalg.norm(b)))
