"""Probe: settings whose trajectories contain rejected steps (reject_if_worse)."""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2505_21404_b200 as P  # noqa: E402

for pname, widths, counts, cap in [
    ("poisson2d", (2, 16, 1), (60, 20), 1e-1),
    ("poisson2d", (2, 8, 8, 1), (80, 20), 1.0),
    ("heat1d", (2, 16, 16, 1), (60, 20, 20), 1e-2),
    ("allen_cahn", (3, 16, 16, 1), (60, 20), 1e-3),
    ("poisson_ball_stde", (10, 16, 1), (40,), 1e3),
]:
    for seed in range(3):
        kw = dict(dim=10, index_set_size=3) if pname == "poisson_ball_stde" else {}
        config = P.OptimizerConfig(max_iters=15, lam_cap=cap, reject_if_worse=True,
                                   deterministic_timing=True)
        tr = P.dngd_run(P.make_problem(pname, **kw), P.MlpSpec(widths), config, seed,
                        counts=counts, init="xavier_normal", track_rel_l2=False)
        rej = [r.iteration for r in tr.rows[1:] if np.isnan(r.eta)]
        print(pname, widths, cap, seed, "rejected at", rej, "aborted", tr.aborted)
