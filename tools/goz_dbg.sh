for d in 0; do DNGD_GOZ_DBG=$d python - <<PY
import sys, numpy as np, torch
sys.path.insert(0,".")
import paper_2505_21404_b200 as P
from paper_2505_21404_b200 import kernels as K
prob = P.make_problem("poisson5d_sin")
spec = P.MlpSpec((5, 512, 512, 512, 512, 1))
rmap = P.PinnResidualMap(prob, spec, prob.sample((3500, 500), np.random.default_rng(0)))
theta = P.xavier_normal_params(spec)
d = rmap._device(); rmap.residuals_act_t(theta); ws = rmap._act_workspace()
Kt = torch.zeros(rmap.m, rmap.m, dtype=torch.float64, device="cuda")
K.gram_factored_act(d["mlp"], d["arr"], d["nclass"], Kt, ws, slices=7); torch.cuda.synchronize()
a=torch.cuda.Event(enable_timing=True); b=torch.cuda.Event(enable_timing=True)
a.record()
for _ in range(3): K.gram_factored_act(d["mlp"], d["arr"], d["nclass"], Kt, ws, slices=7)
b.record(); torch.cuda.synchronize()
print("dbg $d", a.elapsed_time(b)/3, "ms", flush=True)
PY
done
