"""HBM-bound stages with J materialised at a BASELINE config (bench._hbm_stages)."""
import json
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
import bench  # noqa: E402
import paper_2505_21404_b200 as P  # noqa: E402

cfg = bench.CONFIGS[int(sys.argv[1]) if len(sys.argv) > 1 else 3]
prob = P.make_problem(cfg["problem"])
spec = P.MlpSpec(cfg["widths"])
rmap = P.PinnResidualMap(prob, spec, prob.sample(cfg["counts"], np.random.default_rng(0)))
theta = P.xavier_normal_params(spec)
rmap._device()
out = bench._hbm_stages(rmap, theta, 6547.2)
print(json.dumps({k: (v if isinstance(v, str) else {kk: vv for kk, vv in v.items()}) for k, v in out.items()}))
