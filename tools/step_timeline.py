"""Device timeline of bench steps: kernel time vs idle gaps (torch.profiler/CUPTI).

python tools/step_timeline.py [--config 2] [--steps 5]
Prints per-kernel totals and the largest idle gaps with their neighbours."""
import argparse
import collections
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
import paper_2505_21404_b200 as P  # noqa: E402
from paper_2505_21404_b200 import kernels as K  # noqa: E402
from paper_2505_21404_b200.optimizer import _select  # noqa: E402
from paper_2505_21404_b200.solver import fused_dense_step  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--config", type=int, default=2)
ap.add_argument("--steps", type=int, default=5)
a = ap.parse_args()
cfg = bench.CONFIGS[a.config]
problem = P.make_problem(cfg["problem"])
spec = P.MlpSpec(cfg["widths"], seed=0)
rng = np.random.default_rng(1000)
maps = []
base = None
for _ in range(a.steps + 3):
    colloc = P.sample_collocation(problem, cfg["counts"], rng)
    mp = P.PinnResidualMap(problem, spec, colloc) if base is None else base.rebind(colloc)
    mp._device()
    maps.append(mp)
    base = mp
theta = P.xavier_normal_params(spec)
etas = 2.0 ** -np.arange(31, dtype=np.float64)


def step(rmap, theta):
    st, losses, _, loss, _ = fused_dense_step(rmap, theta, None, None, True, 31,
                                              lam_cap=cfg["lam_cap"])
    ls = _select(losses, etas, loss, 31)
    if ls.rejected:
        return theta
    return P.ParameterVector(K.axpby(ls.eta, st.delta.tensor, 1.0, theta.tensor), theta.layout)


for k in range(3):
    theta = step(maps[k], theta)
torch.cuda.synchronize()
from torch.profiler import ProfilerActivity, profile  # noqa: E402

with profile(activities=[ProfilerActivity.CUDA, ProfilerActivity.CPU]) as prof:
    for k in range(a.steps):
        theta = step(maps[3 + k], theta)
    torch.cuda.synchronize()
evs = [e for e in prof.events() if e.device_type.name == "CUDA" and e.device_time_total > 0]
ker = sorted(((e.time_range.start, e.time_range.end, e.name) for e in evs), key=lambda x: x[0])
span = ker[-1][1] - ker[0][0]
busy = sum(e - s for s, e, _ in ker)
print(f"steps {a.steps}: span {span / a.steps:.1f} us/step, kernel busy {busy / a.steps:.1f} us/step, "
      f"launches {len(ker) / a.steps:.0f}/step")
tot = collections.Counter()
cnt = collections.Counter()
for s, e, n in ker:
    tot[n[:70]] += e - s
    cnt[n[:70]] += 1
for n, t in tot.most_common(25):
    print(f"  {t / a.steps:8.1f} us/step  x{cnt[n] / a.steps:5.1f}  {n}")
gaps = collections.Counter()
gapn = collections.Counter()
for (s0, e0, n0), (s1, e1, n1) in zip(ker, ker[1:]):
    g = s1 - max(e0, s0)
    if g > 0:
        key = f"{n0[:40]} -> {n1[:40]}"
        gaps[key] += g
        gapn[key] += 1
print(f"idle total {sum(gaps.values()) / a.steps:.1f} us/step; largest gap sources:")
for k2, g in gaps.most_common(20):
    print(f"  {g / a.steps:8.1f} us/step  x{gapn[k2] / a.steps:5.1f}  {k2}")

# host side: runtime API calls around the largest gaps
cpu = sorted(((e.time_range.start, e.time_range.end, e.name) for e in prof.events()
              if e.device_type.name == "CPU"), key=lambda x: x[0])
big = sorted(((s1 - e0, e0, s1, n0, n1) for (s0, e0, n0), (s1, e1, n1) in zip(ker, ker[1:])
              if s1 - e0 > 40), reverse=True)[:4]
for g, e0, s1, n0, n1 in big:
    print(f"gap {g:.1f} us after {n0[:50]} before {n1[:50]}; host events starting in the window:")
    for s, e, n in cpu:
        if e0 - 150 <= s <= s1:
            print(f"    {s - e0:8.1f} {e - s:8.1f}  {n[:80]}")
