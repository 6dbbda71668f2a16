"""Generate the golden fixtures that pin the CPU oracle to the REAL reference.

Run in the build container only (the reference is not on the GPU box):

    PYTHONPATH=/root/reference/pkg/src python tests/golden/make_golden.py

It imports the unmodified reference package `dngd` from /root/reference,
adds the BASELINE-config pieces the reference lacks (SURVEY §0 G1-G3:
Xavier-normal init, the 3-class 1-D heat problem, the 5-D sine Poisson
problem) as plugins written against the reference's own PdeProblem API
(problems.py:107-146), and records the reference's outputs at reduced
sizes as .npz fixtures next to this script.  Nothing here is imported by
the product package.
"""

from __future__ import annotations

import os
import sys
from dataclasses import replace

import numpy as np

REF = "/root/reference/pkg/src"
if REF not in sys.path:
    sys.path.insert(0, REF)

import dngd  # noqa: E402
import dngd.optimizer as dopt  # noqa: E402
from dngd import ops  # noqa: E402
from dngd.model import IdentityEmbedding, MlpSpec  # noqa: E402
from dngd.params import ParameterVector  # noqa: E402
from dngd.problems import PdeProblem, _box_faces, _box_interior, _cls, _halton, _pairwise_sum  # noqa: E402
from dngd.residuals import BOUNDARY, INITIAL, INTERIOR, CollocationSet, PinnResidualMap  # noqa: E402
from dngd.solver import (  # noqa: E402
    assemble_gramian,
    dense_dual_solve,
    nystrom_build,
    pcg_step,
)

HERE = os.path.dirname(os.path.abspath(__file__))


# -- G1: Xavier-normal init, same layout order as model.py:48-54 -------------------------


def xavier_normal_params(spec: MlpSpec) -> ParameterVector:
    rng = np.random.default_rng(spec.seed)
    arrays = []
    w = spec.layer_widths
    for k in range(len(w) - 1):
        std = np.sqrt(2.0 / (w[k] + w[k + 1]))
        arrays.append(rng.normal(0.0, std, size=(w[k], w[k + 1])))
        arrays.append(np.zeros(w[k + 1]))
    return ParameterVector.from_arrays(arrays, spec.layout())


# -- G2: 1-D heat, three classes ----------------------------------------------------------


class Heat1dThreeClass(PdeProblem):
    name = "heat1d"
    raw_dim = 2
    kappa = 0.1
    default_counts = {INTERIOR: 2000, BOUNDARY: 400, INITIAL: 400}
    default_widths = (2, 64, 64, 64, 64, 1)
    default_lam_cap = 1e-3

    def __init__(self):
        self.embedding = IdentityEmbedding(2)

    def sample(self, counts, rng):
        c = self.resolve_counts(counts)
        pi = _box_interior(rng, c[INTERIOR], [0, 0], [1, 1])
        tb = rng.uniform(size=c[BOUNDARY])
        xb = rng.integers(0, 2, size=c[BOUNDARY]).astype(np.float64)
        x0 = rng.uniform(size=c[INITIAL])
        return CollocationSet(
            [
                _cls(INTERIOR, pi),
                _cls(BOUNDARY, np.column_stack([tb, xb])),
                _cls(INITIAL, np.column_stack([np.zeros(c[INITIAL]), x0])),
            ]
        )

    def class_residual(self, net, cls):
        p = cls.points
        if cls.class_id == INTERIOR:
            jt = net.jet(p, 0)
            jx = net.jet(p, 1)
            return ops.sub(jt.d1, ops.mul(self.kappa, jx.d2))
        return ops.sub(net.u(p), self.exact_solution(p))

    def exact_solution(self, p):
        return np.exp(-self.kappa * np.pi**2 * p[:, 0]) * np.sin(np.pi * p[:, 1])

    def eval_points(self, num=10_000):
        return _halton(num, [0, 0], [1, 1])


# -- G3: d-dimensional sine Poisson -----------------------------------------------------------


class PoissonSin(PdeProblem):
    default_lam_cap = 1e-5

    def __init__(self, dim=5):
        self.dim = dim
        self.name = f"poisson{dim}d_sin"
        self.raw_dim = dim
        self.embedding = IdentityEmbedding(dim)
        self.default_counts = {INTERIOR: 3500, BOUNDARY: 500}
        self.default_widths = (dim, 512, 512, 512, 512, 1)

    def sample(self, counts, rng):
        c = self.resolve_counts(counts)
        d = self.dim
        return CollocationSet(
            [
                _cls(INTERIOR, _box_interior(rng, c[INTERIOR], np.zeros(d), np.ones(d))),
                _cls(BOUNDARY, _box_faces(rng, c[BOUNDARY], np.zeros(d), np.ones(d))),
            ]
        )

    def class_residual(self, net, cls):
        p = cls.points
        if cls.class_id == INTERIOR:
            lap = _pairwise_sum([net.jet(p, j).d2 for j in range(self.dim)])
            f = np.pi**2 * np.sum(np.sin(np.pi * p), axis=1)
            return ops.sub(ops.neg(lap), f)
        return ops.sub(net.u(p), self.exact_solution(p))

    def exact_solution(self, p):
        return np.sum(np.sin(np.pi * p), axis=1)

    def eval_points(self, num=10_000):
        return _halton(num, np.zeros(self.dim), np.ones(self.dim))


# -- fixture writers ----------------------------------------------------------------------------


def _points(colloc):
    out = {f"pts_{c.class_id}": c.points for c in colloc.classes}
    for c in colloc.classes:
        if "stde_idx" in c.aux:
            out[f"idx_{c.class_id}"] = np.asarray(c.aux["stde_idx"])
    return out


def step_fixture(name, problem, widths, counts, seed, lams, store_J_rows=None, probes=3):
    spec = MlpSpec(tuple(widths), seed=seed)
    rng = np.random.default_rng(seed)
    theta = xavier_normal_params(spec)
    colloc = problem.sample(counts, rng)
    rmap = PinnResidualMap(problem, spec, colloc)
    batch, g = rmap.residuals_and_gradient(theta)
    J = rmap.jacobian(theta)
    K = assemble_gramian(rmap, theta).K
    prng = np.random.default_rng(1000 + seed)
    Pn = prng.normal(size=(probes, rmap.n))
    Pm = prng.normal(size=(probes, rmap.m))
    out = dict(
        widths=np.array(widths),
        seed=np.array(seed),
        theta=theta.data,
        r=batch.values,
        g=g,
        K=K,
        probe_n=Pn,
        probe_m=Pm,
        J_probe_n=np.stack([rmap.jvp(theta, p) for p in Pn]),
        JT_probe_m=np.stack([rmap.vjp(theta, p) for p in Pm]),
        J_row_norms=np.linalg.norm(J, axis=1),
        fvv_probe=np.stack([rmap.second_directional(theta, p) for p in Pn]),
        lams=np.array(lams, dtype=np.float64),
        **_points(colloc),
    )
    if store_J_rows is None:
        out["J"] = J
    else:
        out["J_rows_idx"] = np.array(store_J_rows)
        out["J_rows"] = J[store_J_rows]
    for i, lam in enumerate(lams):
        res = dense_dual_solve(rmap, theta, g, lam=lam, use_ga=True)
        plain = dense_dual_solve(rmap, theta, g, lam=lam, use_ga=False)
        v = plain.delta.data
        out[f"v_{i}"] = v
        out[f"delta_{i}"] = res.delta.data
        out[f"ga_ratio_{i}"] = np.array(np.nan if res.ga_ratio is None else res.ga_ratio)
        out[f"lam_used_{i}"] = np.array(res.lambda_used)
        out[f"fvv_{i}"] = rmap.second_directional(theta, v)
        etas = 2.0 ** -np.arange(31, dtype=np.float64)
        cands = theta.data[None, :] + etas[:, None] * res.delta.data[None, :]
        out[f"ls_losses_{i}"] = rmap.loss_many(cands)
    np.savez_compressed(os.path.join(HERE, f"{name}.npz"), **out)
    print(f"wrote {name}: m={rmap.m} n={rmap.n}")


def trajectory_fixture(name, problem, widths, counts, seed, lam_cap, iters, **cfg):
    dopt.init_params = xavier_normal_params  # G1 injection (optimizer.py:17,301)
    spec = MlpSpec(tuple(widths))
    config = dopt.OptimizerConfig(
        max_iters=iters, lam_cap=lam_cap, deterministic_timing=True, **cfg
    )
    trace = dopt.dngd_run(problem, spec, config, seed, counts=counts)
    rows = trace.rows
    out = dict(
        widths=np.array(widths),
        seed=np.array(seed),
        lam_cap=np.array(lam_cap),
        loss=np.array([r.loss for r in rows]),
        rel_l2=np.array([r.rel_l2 for r in rows]),
        lam=np.array([r.lam for r in rows]),
        eta=np.array([r.eta for r in rows]),
        ga_ratio=np.array([r.ga_ratio for r in rows]),
        cg_iterations=np.array([r.cg_iterations for r in rows]),
        final_theta=trace.final_theta.data,
        aborted=np.array(trace.aborted),
    )
    np.savez_compressed(os.path.join(HERE, f"{name}.npz"), **out)
    print(f"wrote {name}: {len(rows)} rows, final loss {rows[-1].loss:.6e}")


def pcg_fixture(name, problem, widths, counts, seed, lam, ell, tol, max_iters):
    spec = MlpSpec(tuple(widths), seed=seed)
    rng = np.random.default_rng(seed)
    theta = xavier_normal_params(spec)
    colloc = problem.sample(counts, rng)
    rmap = PinnResidualMap(problem, spec, colloc)
    _, g = rmap.residuals_and_gradient(theta)
    state = rng.bit_generator.state
    res = pcg_step(rmap, theta, g, lam=lam, landmark_count=ell, tol=tol,
                   max_iters=max_iters, rng=rng)
    rng2 = np.random.default_rng(0)
    rng2.bit_generator.state = state
    P = nystrom_build(rmap, theta, landmark_count=ell, lam=lam, rng=rng2)
    probe = np.random.default_rng(77).normal(size=(3, rmap.m))
    dense = dense_dual_solve(rmap, theta, g, lam=lam, use_ga=False)
    out = dict(
        widths=np.array(widths),
        seed=np.array(seed),
        lam=np.array(lam),
        ell=np.array(ell),
        tol=np.array(tol),
        max_iters=np.array(max_iters),
        theta=theta.data,
        delta=res.delta.data,
        dense_delta=dense.delta.data,
        cg_iterations=np.array(res.cg_iterations),
        landmarks=P.landmarks,
        lam_hat=P.lam_hat,
        probe=probe,
        precond_probe=np.stack([P.apply(p) for p in probe]),
        **_points(colloc),
    )
    np.savez_compressed(os.path.join(HERE, f"{name}.npz"), **out)
    print(f"wrote {name}: iters={res.cg_iterations} rank={P.rank}")


def main():
    from dngd.problems import Poisson2d

    step_fixture("cfg1_step", Poisson2d(), (2, 32, 32, 1), {INTERIOR: 40, BOUNDARY: 16}, 0,
                 [1e-3, 1e-8])
    step_fixture("cfg2_step", Heat1dThreeClass(), (2, 64, 64, 64, 64, 1),
                 {INTERIOR: 24, BOUNDARY: 8, INITIAL: 8}, 1, [1e-3], store_J_rows=[0, 5, 24, 31, 32, 39])
    step_fixture("cfg3_step", PoissonSin(5), (5, 32, 32, 32, 32, 1),
                 {INTERIOR: 24, BOUNDARY: 8}, 2, [1e-5], store_J_rows=[0, 7, 23, 24, 31])
    trajectory_fixture("cfg1_traj", Poisson2d(), (2, 32, 32, 1), {INTERIOR: 90, BOUNDARY: 30},
                       0, 1e-3, 5)
    trajectory_fixture("cfg2_traj", Heat1dThreeClass(), (2, 16, 16, 1),
                       {INTERIOR: 60, BOUNDARY: 20, INITIAL: 20}, 3, 1e-3, 4)
    trajectory_fixture("pcg_traj", Poisson2d(), (2, 16, 16, 1), {INTERIOR: 60, BOUNDARY: 20},
                       4, 1e-3, 3, dense_threshold=10, nystrom_rank=16, cg_max_iters=100)
    pcg_fixture("pcg_step", Poisson2d(), (2, 16, 16, 1), {INTERIOR: 60, BOUNDARY: 20}, 5,
                1e-3, 16, 1e-10, 200)


def main_allen_cahn():
    """Allen-Cahn (problems.py:286-328): periodic embedding + cubic reaction, the
    reference's own problem class, unmodified."""
    from dngd.problems import AllenCahn

    step_fixture("ac_step", AllenCahn(), (3, 32, 32, 32, 1), {INTERIOR: 40, INITIAL: 16}, 6,
                 [1e-3, 1e-6])
    trajectory_fixture("ac_traj", AllenCahn(), (3, 16, 16, 1), {INTERIOR: 60, INITIAL: 20},
                       7, 1e-3, 4)


def main_stde():
    """PoissonBallStde (problems.py:331-402): dirichlet_ball output transform and the
    per-point random Laplacian index subsets, the reference's own problem class."""
    from dngd.problems import PoissonBallStde

    step_fixture("stde_step", PoissonBallStde(10, 3), (10, 16, 16, 1), {INTERIOR: 32}, 8,
                 [1e-3])
    trajectory_fixture("stde_traj", PoissonBallStde(10, 3), (10, 12, 12, 1), {INTERIOR: 40},
                       9, 1e3, 3)
    # wide raw input (din > 12): the device step forms J's input block analytically
    trajectory_fixture("stde_wide_traj", PoissonBallStde(200, 4), (200, 16, 16, 1),
                       {INTERIOR: 48}, 10, 1e3, 3)


def main_ic_shift():
    """ic_shift output transform (model.py:181-277): the reference's own Heat(1) with
    u = phi(t, x) - phi(0, x) + q0(x), q0 = sin(2 pi x) (its exact initial trace)."""
    from dngd.model import OutputTransform
    from dngd.problems import Heat

    class HeatIcShift(Heat):
        def __init__(self):
            super().__init__(1)
            self.name = "heat1d_ic_shift"
            self.transform = OutputTransform(
                "ic_shift", q0=lambda cols: ops.sin(ops.mul(2.0 * np.pi, cols[1])))

    step_fixture("icshift_step", HeatIcShift(), (2, 24, 24, 1), {INTERIOR: 40, BOUNDARY: 16}, 11,
                 [1e-3, 1e-6])
    trajectory_fixture("icshift_traj", HeatIcShift(), (2, 16, 16, 1),
                       {INTERIOR: 60, BOUNDARY: 20}, 12, 1e-3, 4)


if __name__ == "__main__":
    if sys.argv[1:] == ["ic_shift"]:
        main_ic_shift()
    elif sys.argv[1:] == ["allen_cahn"]:
        main_allen_cahn()
    elif sys.argv[1:] == ["stde"]:
        main_stde()
    elif sys.argv[1:] == ["stde_wide"]:
        from dngd.problems import PoissonBallStde
        trajectory_fixture("stde_wide_traj", PoissonBallStde(200, 4), (200, 16, 16, 1),
                           {INTERIOR: 48}, 10, 1e3, 3)
    else:
        main()
        main_allen_cahn()
        main_stde()
        main_ic_shift()
