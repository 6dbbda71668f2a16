"""Pin the numpy oracle to fixtures produced by the unmodified reference.

Fixtures: tests/golden/make_golden.py (imports /root/reference in the build
container).  These run on CPU only.
"""

import os

import numpy as np
import pytest

from oracle import dngd_oracle as O


def _load(golden_dir, name):
    return np.load(os.path.join(golden_dir, f"{name}.npz"))


def _rel(a, b):
    return np.linalg.norm(np.asarray(a) - np.asarray(b)) / max(np.linalg.norm(b), 1e-300)


PROBLEMS = {
    "cfg1_step": (O.OraclePoisson2d(), ("interior", "boundary")),
    "cfg2_step": (O.OracleHeat1d(), ("interior", "boundary", "initial")),
    "cfg3_step": (O.OraclePoissonSin(5), ("interior", "boundary")),
    "ac_step": (O.OracleAllenCahn(), ("interior", "initial")),
    "stde_step": (O.OraclePoissonBallStde(10, 3), ("interior",)),
    "icshift_step": (O.OracleHeatIcShift(), ("interior", "boundary")),
}


def _classes(fx, problem, ids):
    if isinstance(problem, O.OraclePoissonBallStde):
        return problem.classes(fx["pts_interior"], fx["idx_interior"])
    return problem.classes(*[fx[f"pts_{c}"] for c in ids])


@pytest.mark.parametrize("name", sorted(PROBLEMS))
def test_oracle_residuals_jacobian_gram(golden_dir, name):
    fx = _load(golden_dir, name)
    problem, ids = PROBLEMS[name]
    widths = tuple(int(w) for w in fx["widths"])
    classes = _classes(fx, problem, ids)
    theta = O.xavier_normal_init(widths, int(fx["seed"]))
    assert np.array_equal(theta, fx["theta"])  # G1 init bit-identical
    r, J = O.linearize(theta, widths, classes)
    assert _rel(r, fx["r"]) <= 1e-12
    assert _rel(J.T @ r, fx["g"]) <= 1e-11
    if "J" in fx:
        assert _rel(J, fx["J"]) <= 1e-12
    else:
        idx = fx["J_rows_idx"]
        for k, i in enumerate(idx):
            assert _rel(J[i], fx["J_rows"][k]) <= 1e-12
    assert np.max(np.abs(np.linalg.norm(J, axis=1) - fx["J_row_norms"])
                  / np.maximum(fx["J_row_norms"], 1e-300)) <= 1e-12
    K = O.gram(J)
    assert _rel(K, fx["K"]) <= 1e-12
    for p, ref in zip(fx["probe_n"], fx["J_probe_n"]):
        assert _rel(J @ p, ref) <= 1e-11
    for p, ref in zip(fx["probe_m"], fx["JT_probe_m"]):
        assert _rel(J.T @ p, ref) <= 1e-11
    for p, ref in zip(fx["probe_n"], fx["fvv_probe"]):
        assert _rel(O.second_directional(theta, widths, classes, p), ref) <= 1e-10


@pytest.mark.parametrize("name", sorted(PROBLEMS))
def test_oracle_dense_step_and_line_search(golden_dir, name):
    fx = _load(golden_dir, name)
    problem, ids = PROBLEMS[name]
    widths = tuple(int(w) for w in fx["widths"])
    classes = _classes(fx, problem, ids)
    theta = fx["theta"]
    r, J = O.linearize(theta, widths, classes)
    g = J.T @ r
    for i, lam in enumerate(fx["lams"]):
        res = O.dense_dual_solve(J, g, lam, True,
                                 lambda v: O.second_directional(theta, widths, classes, v))
        # floor-relative tolerance: max(1e-8, 10 x oracle self-floor)
        fl = O.direction_floors(J, g, lam,
                                lambda v: O.second_directional(theta, widths, classes, v))
        tol_v = max(1e-8, 10 * fl["v"])
        tol_d = max(1e-8, 10 * fl["delta"])
        assert _rel(res.extras["v"], fx[f"v_{i}"]) <= tol_v
        assert res.lambda_used == fx[f"lam_used_{i}"]
        if not np.isnan(fx[f"ga_ratio_{i}"]):
            assert abs(res.ga_ratio - fx[f"ga_ratio_{i}"]) <= tol_v * max(1.0, fx[f"ga_ratio_{i}"])
        assert _rel(res.delta, fx[f"delta_{i}"]) <= tol_d
        fvv = O.second_directional(theta, widths, classes, fx[f"v_{i}"])
        assert _rel(fvv, fx[f"fvv_{i}"]) <= 1e-10
        etas = 2.0 ** -np.arange(31, dtype=np.float64)
        cands = theta[None, :] + etas[:, None] * fx[f"delta_{i}"][None, :]
        losses = O.loss_many(cands, widths, classes)
        np.testing.assert_allclose(losses, fx[f"ls_losses_{i}"], rtol=1e-10)


TRAJ = {
    "cfg1_traj": (O.OraclePoisson2d(), (90, 30), O.LoopConfig(lam_cap=1e-3, max_iters=5)),
    "cfg2_traj": (O.OracleHeat1d(), (60, 20, 20), O.LoopConfig(lam_cap=1e-3, max_iters=4)),
    "ac_traj": (O.OracleAllenCahn(), (60, 20), O.LoopConfig(lam_cap=1e-3, max_iters=4)),
    "stde_traj": (O.OraclePoissonBallStde(10, 3), (40,), O.LoopConfig(lam_cap=1e3, max_iters=3)),
    "stde_wide_traj": (O.OraclePoissonBallStde(200, 4), (48,),
                       O.LoopConfig(lam_cap=1e3, max_iters=3)),
    "icshift_traj": (O.OracleHeatIcShift(), (60, 20), O.LoopConfig(lam_cap=1e-3, max_iters=4)),
    "pcg_traj": (O.OraclePoisson2d(), (60, 20),
                 O.LoopConfig(lam_cap=1e-3, max_iters=3, dense_threshold=10, nystrom_rank=16,
                              cg_max_iters=100)),
}


REL_L2 = {"cfg1_traj": "poisson2d", "cfg2_traj": "heat1d", "pcg_traj": "poisson2d"}


@pytest.mark.parametrize("name", sorted(TRAJ))
def test_oracle_trajectory(golden_dir, name):
    fx = _load(golden_dir, name)
    problem, counts, cfg = TRAJ[name]
    widths = tuple(int(w) for w in fx["widths"])
    rel = None
    if name in REL_L2:  # the oracle's rel-L2 metric on the problem's evaluation grid
        from paper_2505_21404_b200.problems import make_problem

        prob = make_problem(REL_L2[name])
        pts = prob.eval_points()
        rel = O.rel_l2_fn(widths, pts, prob.exact_solution(pts))
    rows, theta = O.dngd_run(problem, widths, counts, cfg, int(fx["seed"]), rel_l2=rel)
    losses = np.array([r["loss"] for r in rows])
    np.testing.assert_allclose(losses, fx["loss"], rtol=1e-6)
    if rel is not None:
        np.testing.assert_allclose([r["rel_l2"] for r in rows], fx["rel_l2"], rtol=1e-6)
    etas = np.array([r["eta"] for r in rows])
    np.testing.assert_array_equal(etas[1:], fx["eta"][1:])
    np.testing.assert_allclose([r["lam"] for r in rows][1:], fx["lam"][1:], rtol=1e-6)
    # CG stops at |r| <= 1e-10 |b|, at the rounding floor: allow one iteration either way
    its = np.array([r["cg_iterations"] for r in rows])
    assert np.max(np.abs(its - fx["cg_iterations"])) <= 1
    assert _rel(theta, fx["final_theta"]) <= 1e-6


def test_oracle_pcg_and_nystrom(golden_dir):
    fx = _load(golden_dir, "pcg_step")
    problem = O.OraclePoisson2d()
    widths = tuple(int(w) for w in fx["widths"])
    seed = int(fx["seed"])
    rng = np.random.default_rng(seed)
    classes = problem.sample((60, 20), rng)
    np.testing.assert_array_equal(classes[0].points, fx["pts_interior"])
    theta = fx["theta"]
    r, J = O.linearize(theta, widths, classes)
    g = J.T @ r
    lam, ell = float(fx["lam"]), int(fx["ell"])
    state = rng.bit_generator.state
    res = O.pcg_step(J, g, lam, ell, float(fx["tol"]), int(fx["max_iters"]), rng)
    assert res.cg_iterations == int(fx["cg_iterations"])
    assert _rel(res.delta, fx["delta"]) <= 1e-6
    rng2 = np.random.default_rng(0)
    rng2.bit_generator.state = state
    P = O.nystrom_build(J, ell, lam, rng2)
    np.testing.assert_array_equal(P.landmarks, fx["landmarks"])
    np.testing.assert_allclose(P.lam_hat, fx["lam_hat"], rtol=1e-8, atol=1e-12 * fx["lam_hat"][0])
    for p, ref in zip(fx["probe"], fx["precond_probe"]):
        assert _rel(P.apply(p), ref) <= 1e-8


def test_oracle_known_answers():
    # param counts (model.py:44-46)
    assert O.param_count((2, 32, 32, 1)) == 1185
    assert O.param_count((2, 64, 64, 64, 64, 1)) == 12737
    assert O.param_count((5, 512, 512, 512, 512, 1)) == 791553
    assert O.param_count((5, 1792, 1792, 1792, 1792, 1792, 1)) == 12864769
    assert O.param_count((2, 256, 256, 256, 256, 1)) == 198401
    # damping table (test_optimizer.py:43-57)
    assert O.lm_damping(0.3, 1e-5) == 1e-5
    assert O.lm_damping(1e-7, 1e-5) == 1e-7
    assert O.lm_damping(0.0, 1e-5) == 1e-12
    # identity J closed form (test_solver.py:136-145)
    rng = np.random.default_rng(4)
    c = rng.normal(size=6)
    th = rng.normal(size=6)
    r = th + c
    res = O.dense_dual_solve(np.eye(6), r, 0.25, use_ga=False)
    assert np.allclose(res.delta, -r / 1.25, atol=1e-12)
    # Cholesky retry ladder (test_solver.py:206-211)
    _, lam = O.chol_with_retries(-np.eye(3), 1e-3)
    assert lam == pytest.approx(10.0)
    with pytest.raises(O.OracleFactorizationError):
        O.chol_with_retries(-np.eye(3), 1e-12)


def test_exact_solutions_annihilate_residuals():
    """Exact-solution residual check for the G2/G3 plugins (test_problems.py:40-66 style),
    using second-order finite differences of u* inside the operator definition."""
    rng = np.random.default_rng(0)
    for prob in (O.OracleHeat1d(), O.OraclePoissonSin(5)):
        if isinstance(prob, O.OracleHeat1d):
            classes = prob.sample((50, 20, 20), rng)
        else:
            classes = prob.sample((50, 20), rng)
        for cls in classes:
            p = cls.points
            h = 1e-4
            u = prob.exact(p)
            val = cls.cu * u - cls.f
            for j, cg in zip(cls.grad_dims, cls.cg):
                e = np.zeros(p.shape[1]); e[j] = h
                val = val + cg * (prob.exact(p + e) - prob.exact(p - e)) / (2 * h)
            for j in cls.lap_dims:
                e = np.zeros(p.shape[1]); e[j] = h
                val = val + cls.cl * (prob.exact(p + e) - 2 * u + prob.exact(p - e)) / h**2
            assert np.max(np.abs(val)) <= 1e-5 * max(1.0, np.max(np.abs(cls.f)))
