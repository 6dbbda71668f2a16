"""Kernel breakdown of one config-3 J^T w from the activations (CUPTI via torch.profiler)."""
import collections
import os
import sys

import numpy as np
import torch
from torch.profiler import ProfilerActivity, profile

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2505_21404_b200 as P  # noqa: E402

prob = P.make_problem("poisson5d_sin")
spec = P.MlpSpec((5, 512, 512, 512, 512, 1))
rmap = P.PinnResidualMap(prob, spec, prob.sample((3500, 500), np.random.default_rng(0)))
theta = P.xavier_normal_params(spec)
rmap.residuals_act_t(theta)  # activations only: J is never materialised (the product path)
w = torch.randn(rmap.m, dtype=torch.float64, device="cuda")
f = lambda: rmap.vjp_t(theta, w)  # noqa: E731
for _ in range(2):
    f()
torch.cuda.synchronize()
a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
a.record()
for _ in range(5):
    f()
b.record()
torch.cuda.synchronize()
print(f"J^T w {a.elapsed_time(b) / 5:.3f} ms (events)")
with profile(activities=[ProfilerActivity.CUDA]) as prof:
    f()
    torch.cuda.synchronize()
agg = collections.defaultdict(lambda: [0, 0.0])
for ev in prof.events():
    if ev.device_type == torch.autograd.DeviceType.CUDA:
        k = ev.name.split("(")[0][:70]
        agg[k][0] += 1
        agg[k][1] += ev.device_time_total
tot = sum(v[1] for v in agg.values())
for k, (n, t) in sorted(agg.items(), key=lambda x: -x[1][1]):
    print(f"{n:4d} {t / 1e3:9.3f} ms {100 * t / tot:5.1f}%  {k}")
