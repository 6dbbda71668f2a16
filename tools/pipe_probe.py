"""Probe: pipelined vs eager loop on settings that trigger factorisation failures
and rejections (used to pick the parity-test cases)."""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2505_21404_b200 as P  # noqa: E402


def run(pname, widths, counts, pipe, **cfg):
    if pipe:
        os.environ.pop("DNGD_NO_PIPELINE", None)
    else:
        os.environ["DNGD_NO_PIPELINE"] = "1"
    config = P.OptimizerConfig(deterministic_timing=True, **cfg)
    return P.dngd_run(P.make_problem(pname), P.MlpSpec(widths), config, 3, counts=counts,
                      init="xavier_normal")


for pname, widths, counts, cfg in [
    ("poisson2d", (2, 4, 1), (200, 50), dict(max_iters=12, lam_cap=1e-12)),
    ("poisson2d", (2, 3, 1), (300, 60), dict(max_iters=12, lam_cap=1e-12, reject_if_worse=True)),
    ("heat1d", (2, 8, 8, 1), (200, 40, 40), dict(max_iters=12, lam_cap=1e-12, reject_if_worse=True)),
]:
    a = run(pname, widths, counts, False, **cfg)
    b = run(pname, widths, counts, True, **cfg)
    print(pname, widths, "aborted", a.aborted, b.aborted, a.abort_reason, b.abort_reason)
    for ra, rb in zip(a.rows, b.rows):
        print(f"  {ra.iteration:3d} {ra.loss:.6e} {rb.loss:.6e} lam {ra.lam:.1e} {rb.lam:.1e} eta {ra.eta} {rb.eta} rel {ra.rel_l2:.4e} {rb.rel_l2:.4e}")
    print("  rows", len(a.rows), len(b.rows), "theta diff",
          float(np.max(np.abs(a.final_theta.data - b.final_theta.data))))
