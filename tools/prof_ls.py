"""Kernel breakdown of one config-3 31-candidate line search (CUPTI via torch.profiler,
concurrent timing -- not ncu's serialised replay): what the stage spends its time on."""
import collections
import os
import sys

import numpy as np
import torch
from torch.profiler import ProfilerActivity, profile

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2505_21404_b200 as P  # noqa: E402

widths = tuple(int(x) for x in sys.argv[1].split(",")) if len(sys.argv) > 1 else (5, 512, 512, 512, 512, 1)
counts = tuple(int(x) for x in sys.argv[2].split(",")) if len(sys.argv) > 2 else (3500, 500)
if os.environ.get("LS_BUDGET_GB"):  # line-search activation chunk budget (experiment)
    P.PinnResidualMap.LOSS_WS_BUDGET = int(float(os.environ["LS_BUDGET_GB"]) * 2**30)
prob = P.make_problem(sys.argv[3] if len(sys.argv) > 3 else "poisson5d_sin")
spec = P.MlpSpec(widths)
rmap = P.PinnResidualMap(prob, spec, prob.sample(counts, np.random.default_rng(0)))
theta = P.xavier_normal_params(spec)
delta = torch.randn(spec.param_count(), dtype=torch.float64, device="cuda") * 1e-3
etas = torch.as_tensor(2.0 ** -np.arange(31), device="cuda")
for _ in range(2):
    rmap.losses_along_t(theta, delta, etas)
torch.cuda.synchronize()
a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
a.record()
for _ in range(3):
    rmap.losses_along_t(theta, delta, etas)
b.record()
torch.cuda.synchronize()
print(f"line search {a.elapsed_time(b) / 3:.2f} ms (events)")
with profile(activities=[ProfilerActivity.CUDA]) as prof:
    rmap.losses_along_t(theta, delta, etas)
    torch.cuda.synchronize()
agg = collections.defaultdict(lambda: [0, 0.0])
for ev in prof.events():
    if ev.device_type == torch.autograd.DeviceType.CUDA:
        k = ev.name.split("(")[0][:70]
        agg[k][0] += 1
        agg[k][1] += ev.device_time_total if hasattr(ev, "device_time_total") else ev.cuda_time_total
tot = sum(v[1] for v in agg.values())
for k, (n, t) in sorted(agg.items(), key=lambda x: -x[1][1]):
    print(f"{n:4d} {t / 1e3:9.3f} ms {100 * t / tot:5.1f}%  {k}")
