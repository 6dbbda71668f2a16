"""Kernel breakdown of one device stage at a BASELINE config (CUPTI via torch.profiler):
  python tools/prof_stage.py {ls|vjp|jvp|fvv|act} [config 3|4|5]"""
import collections
import os
import sys

import numpy as np
import torch
from torch.profiler import ProfilerActivity, profile

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2505_21404_b200 as P  # noqa: E402

stage = sys.argv[1] if len(sys.argv) > 1 else "fvv"
cfg = int(sys.argv[2]) if len(sys.argv) > 2 else 3
widths, counts, pname = {3: ((5, 512, 512, 512, 512, 1), (3500, 500), "poisson5d_sin"),
                         4: ((5, 1792, 1792, 1792, 1792, 1792, 1), (7000, 1000), "poisson5d_sin"),
                         5: ((2, 256, 256, 256, 256, 1), (30000, 2000), "poisson2d")}[cfg]
prob = P.make_problem(pname)
spec = P.MlpSpec(widths)
rmap = P.PinnResidualMap(prob, spec, prob.sample(counts, np.random.default_rng(0)))
theta = P.xavier_normal_params(spec)
rmap.residuals_act_t(theta)
dev = torch.randn(spec.param_count(), dtype=torch.float64, device="cuda") * 1e-3
etas = torch.as_tensor(2.0 ** -np.arange(31), device="cuda")
wv = torch.randn(rmap.m, dtype=torch.float64, device="cuda")
fn = {"ls": lambda: rmap.losses_along_t(theta, dev, etas),
      "vjp": lambda: rmap.vjp_t(theta, wv),
      "fvv": lambda: rmap.fvv_t(theta, dev),
      "jvp": lambda: rmap.jvp_t(theta, dev),
      "act": lambda: (rmap._invalidate() if hasattr(rmap, "_invalidate") else None,
                      rmap.residuals_act_t(P.ParameterVector(theta.data + 0.0, spec.layout())))}[stage]
for _ in range(2):
    fn()
torch.cuda.synchronize()
a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
a.record()
for _ in range(3):
    fn()
b.record()
torch.cuda.synchronize()
print(f"{stage} config {cfg}: {a.elapsed_time(b) / 3:.3f} ms (events)")
with profile(activities=[ProfilerActivity.CUDA]) as prof:
    fn()
    torch.cuda.synchronize()
agg = collections.defaultdict(lambda: [0, 0.0])
for ev in prof.events():
    if ev.device_type == torch.autograd.DeviceType.CUDA:
        k = ev.name.split("(")[0][:70]
        agg[k][0] += 1
        agg[k][1] += ev.device_time_total
tot = sum(v[1] for v in agg.values())
for k, (n, t) in sorted(agg.items(), key=lambda x: -x[1][1])[:14]:
    print(f"{n:4d} {t / 1e3:9.3f} ms {100 * t / tot:5.1f}%  {k}")
