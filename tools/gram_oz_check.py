"""Emulated-FP64 (int8 Ozaki) factored Gram vs the FP64 DMMA factored Gram on the
BASELINE shapes: accuracy (max and Frobenius relative difference, and vs the
materialised J J^T where it fits) and CUDA-event kernel time."""
import json
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2505_21404_b200 as P  # noqa: E402
from paper_2505_21404_b200 import kernels as K  # noqa: E402

CASES = [("heat1d", (2, 64, 64, 64, 64, 1), (2000, 400, 400)),
         ("poisson5d_sin", (5, 128, 128, 128, 128, 1), (3500, 500)),
         ("poisson5d_sin", (5, 512, 512, 512, 512, 1), (3500, 500))]
if len(sys.argv) > 1 and sys.argv[1] == "c3":
    CASES = CASES[2:]
if len(sys.argv) > 1 and sys.argv[1] == "cfg4":
    CASES = [("poisson5d_sin", (5, 1792, 1792, 1792, 1792, 1792, 1), (7000, 1000))]


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
    rmap.residuals_act_t(theta)
    ws = rmap._act_workspace()
    out = {"case": name, "widths": widths, "m": m, "n": rmap.n}
    Ks = {}
    for s in (0, 6, 7):
        Kt = torch.zeros(m, m, dtype=torch.float64, device="cuda")
        out[f"ms_s{s}"] = timed(lambda: K.gram_factored_act(d["mlp"], d["arr"], d["nclass"], Kt, ws, slices=s))
        Ks[s] = Kt
    ref = Ks[0]
    nrm = float(ref.norm())
    for s in (6, 7):
        dK = Ks[s] - ref
        out[f"rel_fro_s{s}"] = float(dK.norm()) / nrm
        out[f"rel_max_s{s}"] = float(dK.abs().max() / ref.abs().max())
        out[f"sym_s{s}"] = float((Ks[s] - Ks[s].T).abs().max())
    if rmap.n * m * 8 < 30e9:
        rmap._cache = None
        _, J = rmap.linearize_t(theta)
        Km = K.syrk(J, rmap.n)
        torch.cuda.synchronize()
        for s in (0, 6, 7):
            out[f"vs_JJt_s{s}"] = float((Ks[s] - Km).norm()) / float(Km.norm())
        del J, Km
    print(json.dumps(out), flush=True)
    del Ks, ref
    torch.cuda.empty_cache()
