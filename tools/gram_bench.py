"""Time the factored Gram (no J) against assemble(J) + SYRK on the config shapes."""
import json
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2505_21404_b200 as P  # noqa: E402
from paper_2505_21404_b200 import kernels as K  # noqa: E402

CASES = [("poisson2d", (2, 32, 32, 1), (900, 120)),
         ("heat1d", (2, 64, 64, 64, 64, 1), (2000, 400, 400)),
         ("poisson5d_sin", (5, 512, 512, 512, 512, 1), (3500, 500))]


def timed(fn, iters=3):
    fn()
    torch.cuda.synchronize()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    for _ in range(iters):
        fn()
    e.record()
    torch.cuda.synchronize()
    return s.elapsed_time(e) / iters


for name, widths, counts in CASES:
    prob = P.make_problem(name)
    spec = P.MlpSpec(widths)
    rmap = P.PinnResidualMap(prob, spec, prob.sample(counts, np.random.default_rng(0)))
    theta = P.xavier_normal_params(spec)
    d = rmap._device()
    m = rmap.m
    r = torch.empty(m, dtype=torch.float64, device="cuda")
    Kf = torch.empty(m, m, dtype=torch.float64, device="cuda")
    ws = K.workspace("pinn", d["ws_bytes"])
    th = theta.tensor

    def fact():
        K.gram_factored(d["mlp"], th, d["arr"], d["nclass"], r, Kf, ws)

    def mat():
        rmap._cache = None
        _, J = rmap.linearize_t(theta)
        return K.syrk(J, rmap.n)

    t_f = timed(fact)
    t_m = timed(mat)
    Km = mat()
    torch.cuda.synchronize()
    rel = float((Kf - Km).norm() / Km.norm())
    print(json.dumps({"case": name, "m": m, "n": rmap.n, "factored_ms": t_f,
                      "assemble_plus_syrk_ms": t_m, "speedup": t_m / t_f, "rel_diff": rel}),
          flush=True)
