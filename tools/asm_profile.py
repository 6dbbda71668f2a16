"""Per-kernel durations of one J assembly (dngd_assemble) at the bench config:
python tools/asm_profile.py [config]."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
from paper_2505_21404_b200 import kernels as K  # noqa: E402

cfgno = int(sys.argv[1]) if len(sys.argv) > 1 else 2
cfg = bench.CONFIGS[cfgno]
import numpy as np  # noqa: E402

import paper_2505_21404_b200 as P  # noqa: E402

problem = P.make_problem(cfg["problem"], **cfg.get("problem_kw", {}))
spec = P.MlpSpec(cfg["widths"], seed=0)
rmap = P.PinnResidualMap(problem, spec, P.sample_collocation(problem, cfg["counts"],
                                                            np.random.default_rng(1000)))
from paper_2505_21404_b200.model import init_params  # noqa: E402

theta = init_params(spec)
th = rmap._theta_t(theta)
d = rmap._device()
m, n = rmap.m, rmap.n
J = torch.empty((m, K.pad_ld(n)), dtype=torch.float64, device="cuda")
r = torch.empty(m, dtype=torch.float64, device="cuda")
ws = rmap._act_workspace()
for _ in range(3):
    K.assemble(d["mlp"], th, d["arr"], d["nclass"], r, J, 0, n, ws)
torch.cuda.synchronize()
from torch.profiler import ProfilerActivity, profile  # noqa: E402

with profile(activities=[ProfilerActivity.CUDA]) as prof:
    K.assemble(d["mlp"], th, d["arr"], d["nclass"], r, J, 0, n, ws)
    torch.cuda.synchronize()
evs = sorted((e for e in prof.events() if e.device_type.name == "CUDA"), key=lambda e: e.time_range.start)
t0 = evs[0].time_range.start
tot = {}
for e in evs:
    dur = e.time_range.end - e.time_range.start
    print(f"{e.time_range.start - t0:9.1f} {dur:7.1f}  {e.name[:70]}")
    tot[e.name[:40]] = tot.get(e.name[:40], 0) + dur
print("span", evs[-1].time_range.end - t0, "us;  J bytes", 8 * m * n)
for k, v in sorted(tot.items(), key=lambda x: -x[1]):
    print(f"{v:8.1f} {k}")
