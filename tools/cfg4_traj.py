import sys, numpy as np
sys.path.insert(0, ".")
import paper_2505_21404_b200 as P
cfg = P.OptimizerConfig(max_iters=8, lam_cap=1e-5, deterministic_timing=True)
tr = P.dngd_run(P.make_problem("poisson5d_sin"), P.MlpSpec((5,1792,1792,1792,1792,1792,1)), cfg, 0,
                counts=(7000, 1000), init="xavier_normal")
for r in tr.rows: print(r.iteration, r.loss, r.eta, r.lam, getattr(r, "ga_ratio", None))
print("aborted", tr.aborted, tr.abort_reason)
