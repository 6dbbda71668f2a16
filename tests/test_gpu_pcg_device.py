"""The hand-written Nystrom numerics and the device-resident CG loop (reference
solver.py:237-366): the Jacobi eigensolver against numpy's eigh, the sketch-form
preconditioner against the reference's (U, lam_hat) form, and the graph-resident
CG loop against the host-driven loop on the same operator."""

import numpy as np
import pytest

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")


@pytest.fixture(scope="module")
def P():
    if not torch.cuda.is_available():
        pytest.skip("needs CUDA")
    import paper_2505_21404_b200 as P
    return P


def _psd(n, rank, seed, spread=1e8):
    rng = np.random.default_rng(seed)
    Q, _ = np.linalg.qr(rng.normal(size=(n, n)))
    ev = np.zeros(n)
    ev[:rank] = np.logspace(0, -np.log10(spread), rank)
    return (Q * ev) @ Q.T


@pytest.mark.parametrize("n,kind", [(1, "rand"), (2, "rand"), (3, "rand"), (17, "rand"),
                                    (64, "psd"), (255, "psd_lowrank"), (512, "psd"),
                                    (512, "psd_lowrank"), (96, "degenerate")])
def test_jacobi_eigensolver_matches_eigh(P, n, kind):
    from paper_2505_21404_b200 import kernels as K

    rng = np.random.default_rng(n)
    if kind == "rand":  # PSD (the solver returns |lambda|: K_II is a Gram block)
        A = rng.normal(size=(n, n))
        A = A @ A.T
    elif kind == "psd":
        A = _psd(n, n, n)
    elif kind == "psd_lowrank":
        A = _psd(n, n // 3, n)
    else:  # repeated eigenvalues
        Q, _ = np.linalg.qr(rng.normal(size=(n, n)))
        ev = np.repeat([3.0, 1.0, 0.0], n // 3)
        A = (Q * ev) @ Q.T
    A = 0.5 * (A + A.T)
    At = torch.zeros((n, K.pad_ld(n, 2)), dtype=torch.float64, device="cuda")
    At[:, :n] = torch.as_tensor(A, device="cuda")
    w, V, sweeps = K.syev_jacobi(At[:, :n], n)
    w, V = w.cpu().numpy(), V.cpu().numpy()
    ref = np.linalg.eigvalsh(A)
    scale = max(np.abs(ref).max(), 1e-300)
    np.testing.assert_allclose(np.sort(w), np.abs(ref) if kind == 'psd_lowrank' else ref,
                               atol=1e-12 * scale, rtol=0)
    big = w >= 0.0  # accumulated rotations: orthogonal to rounding
    Vb = V[:, big]
    assert np.linalg.norm(Vb.T @ Vb - np.eye(int(big.sum()))) <= 1e-12 * n
    assert np.linalg.norm(A - (V * w) @ V.T) <= 1e-12 * max(np.linalg.norm(A), 1e-300)
    floor = 1e-10 * ref[-1]  # the preconditioner's decision is exact
    assert int((w > floor).sum()) == int((ref > floor).sum())
    assert 1 <= int(sweeps.item()) <= 60  # converged (a sweep with no rotation)


def test_sketch_preconditioner_equals_reference_form(P):
    """P^-1 v of the sketch form == U (lam_hat + lam)^-1 U^T v + (v - U U^T v)/lam
    built from the same sketch by an SVD (solver.py:74-83, 262-277)."""
    from paper_2505_21404_b200.solver import NystromPreconditioner, nystrom_from_columns

    rng = np.random.default_rng(0)
    m, n, ell, lam = 300, 80, 40, 1e-3
    Jm = rng.normal(size=(m, n)) * np.logspace(0, -6, n)
    Kfull = Jm @ Jm.T
    landmarks = np.sort(rng.choice(m, size=ell, replace=False))
    Kc = torch.as_tensor(np.ascontiguousarray(Kfull[:, landmarks]), device="cuda")
    pre = nystrom_from_columns(Kc, landmarks, lam)
    # the reference numerics in numpy
    K_II = 0.5 * (Kfull[np.ix_(landmarks, landmarks)] + Kfull[np.ix_(landmarks, landmarks)].T)
    ev, Q = np.linalg.eigh(K_II)
    keep = ev > 1e-10 * max(ev[-1], 0.0)
    lq, Q = ev[keep][::-1], Q[:, keep][:, ::-1]
    Ut = Kfull[:, landmarks] @ Q / lq
    Ut[landmarks] = Q
    U, S, _ = np.linalg.svd(Ut * np.sqrt(lq), full_matrices=False)
    ref = NystromPreconditioner(U, S**2, lam, landmarks)
    assert pre.rank == int(keep.sum())
    for _ in range(4):
        v = rng.normal(size=m)
        a, b = pre.apply(v), ref.apply(v)
        assert np.linalg.norm(a - b) <= 1e-9 * np.linalg.norm(b)
    np.testing.assert_allclose(pre.lam_hat, S**2, rtol=1e-8, atol=1e-12 * S[0] ** 2)


@pytest.mark.parametrize("jfree", [False, True])
def test_device_cg_loop_matches_host_loop(P, jfree):
    """The graph-resident loop (one launch, WHILE node) and the host-driven loop
    (solver.cg_iterate) on the same operator, preconditioner and tolerance:
    same iteration count, same iterate to rounding."""
    from paper_2505_21404_b200.solver import DeviceCG, cg_iterate

    prob = P.make_problem("poisson2d")
    spec = P.MlpSpec((2, 24, 24, 1))
    rmap = P.PinnResidualMap(prob, spec, prob.sample((400, 80), np.random.default_rng(1)))
    if jfree:
        rmap.gram_mode = "factored"
    theta = P.xavier_normal_params(spec)
    _, g = rmap.residuals_and_gradient(theta)
    lam = 1e-4
    for tol, iters in ((1e-10, 200), (1e-14, 7)):  # converged; stopped by the cap
        outs = []
        for device_loop in (True, False):
            res = P.pcg_step(rmap, theta, None if jfree else g, lam=lam, landmark_count=20,
                             tol=tol, max_iters=iters, rng=np.random.default_rng(5))
            outs.append(res)
            if device_loop:
                import paper_2505_21404_b200.solver as S

                orig = S.DeviceCG.solve

                def host_solve(self, apply_A, precond, b, tol_, max_iters_, keyfn):
                    from paper_2505_21404_b200.solver import _alloc_apply

                    return cg_iterate(lambda p: _alloc_apply(apply_A, p), precond, b,
                                      float(b.norm().item()), tol_, max_iters_)

                S.DeviceCG.solve = host_solve
        S.DeviceCG.solve = orig
        dev, host = outs
        assert dev.cg_iterations == host.cg_iterations
        assert dev.warning == host.warning
        d, h = dev.delta.data, host.delta.data
        assert np.linalg.norm(d - h) <= 1e-8 * np.linalg.norm(h)
