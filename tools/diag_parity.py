"""Diagnose GPU-vs-reference direction differences at small lambda (cfg1_step fixture)."""
import os, sys
import numpy as np, scipy.linalg, torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2505_21404_b200 as P
from paper_2505_21404_b200 import kernels as K

rel = lambda a, b: float(np.linalg.norm(a - b) / np.linalg.norm(b))
fx = np.load("tests/golden/cfg1_step.npz")
prob = P.make_problem("poisson2d")
spec = P.MlpSpec((2, 32, 32, 1))
cs = P.CollocationSet([P.CollocationClass(c, fx[f"pts_{c}"], 1 / np.sqrt(len(fx[f"pts_{c}"])))
                       for c in ("interior", "boundary")])
rmap = P.PinnResidualMap(prob, spec, cs)
th = P.ParameterVector(fx["theta"], spec.layout())
Jg = rmap.jacobian(th)
Jr = fx["J"]
print("J rel", rel(Jg, Jr), "max abs", np.abs(Jg - Jr).max())
Kg = P.assemble_gramian(rmap, th).K
Kr = fx["K"]
print("K rel", rel(Kg, Kr), "K(Jr)np rel", rel(Jr @ Jr.T, Kr))
Jd = torch.zeros((Jr.shape[0], K.pad_ld(Jr.shape[1])), dtype=torch.float64, device="cuda")
Jd[:, :Jr.shape[1]] = torch.as_tensor(Jr, device="cuda")
Kgr = K.syrk(Jd, Jr.shape[1]).cpu().numpy()
print("syrk(J_ref) vs K_ref", rel(Kgr, Kr))
g = Jr.T @ fx["r"]
m = Kr.shape[0]
for lam in (1e-3, 1e-8):
    b = -(Jr @ g)
    yr = scipy.linalg.cho_solve(scipy.linalg.cho_factor(Kr + lam * np.eye(m), lower=True), b)
    fac = K.CholeskyFactor(m, "cuda")
    fac.factor(torch.as_tensor(Kr, device="cuda"), lam)
    bd = torch.as_tensor(b, device="cuda").clone()
    fac.solve_(bd)
    yg = bd.cpu().numpy()
    L = np.tril(fac.L[:, :m].cpu().numpy())
    Lr = np.linalg.cholesky(Kr + lam * np.eye(m))
    be = np.linalg.norm((Kr + lam * np.eye(m)) @ yg - b) / (np.linalg.norm(Kr) * np.linalg.norm(yg))
    ber = np.linalg.norm((Kr + lam * np.eye(m)) @ yr - b) / (np.linalg.norm(Kr) * np.linalg.norm(yr))
    print(f"lam {lam}: L rel {rel(L, Lr):.2e} y rel {rel(yg, yr):.2e} bwd err gpu {be:.2e} ref {ber:.2e}")
    vr = -(Jr.T @ yr + g) / lam
    vg = -(Jr.T @ yg + g) / lam
    print("   v from gpu potrs (ref K):", rel(vg, vr))
    # our K with numpy solve
    yk = scipy.linalg.cho_solve(scipy.linalg.cho_factor(Kg + lam * np.eye(m), lower=True), b)
    print("   v from numpy solve on gpu K:", rel(-(Jr.T @ yk + g) / lam, vr))
