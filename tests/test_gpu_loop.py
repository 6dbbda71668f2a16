"""The pipelined dense loop (device-side line-search selection, theta update and
rejection multiplier; iteration i+1 queued before iteration i is read back) against
the step-by-step loop and the host selection rules of optimizer.py:148-166 /
226-247."""

import math

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


def _host_rules(losses, etas, rr, info, anyd, reject_if_worse, mult):
    """The eager loop's decisions (optimizer._select + the accept/reject test)."""
    loss = 0.5 * rr
    if not math.isfinite(loss):
        return 3, None, None, mult
    if info != 0:
        return 2, None, None, mult
    if not anyd:
        return 0, 1.0, loss, 1.0
    finite = np.isfinite(losses)
    if not finite.any():
        return 1, None, None, mult * 10.0
    j = int(np.argmin(np.where(finite, losses, np.inf)))
    if reject_if_worse and losses[j] > loss:
        return 1, None, None, mult * 10.0
    return 0, float(etas[j]), float(losses[j]), 1.0


def test_ls_select_matches_host_rules(P):
    from paper_2505_21404_b200 import kernels as K

    rng = np.random.default_rng(0)
    etas = 2.0 ** -np.arange(31, dtype=np.float64)
    et = torch.as_tensor(etas, device="cuda")
    cases = []
    for k in range(300):
        losses = rng.uniform(0.5, 2.0, size=31)
        kind = k % 10
        if kind == 1:
            losses[rng.integers(0, 31, size=5)] = np.nan
        elif kind == 2:
            losses[:] = np.nan
        elif kind == 3:
            losses[rng.integers(0, 31, size=4)] = np.inf
        elif kind == 4:  # ties: the larger eta wins
            losses[7] = losses[19] = losses.min() - 0.1
        elif kind == 5:
            losses[:] = 3.0  # all worse than the current loss
        rr = 2.0 * rng.uniform(0.8, 1.5)
        if kind == 6:
            rr = np.nan
        info = 5 if kind == 7 else 0
        anyd = 0.0 if kind == 8 else 1.0
        cases.append((losses, rr, info, anyd, bool(k % 3 == 0), 10.0 ** (k % 4)))
    for losses, rr, info, anyd, riw, mult in cases:
        sel = torch.zeros(4, dtype=torch.float64, device="cuda")
        m = torch.tensor([mult], dtype=torch.float64, device="cuda")
        K.ls_select(torch.as_tensor(losses, device="cuda"), et,
                    torch.tensor([rr], dtype=torch.float64, device="cuda"),
                    torch.tensor([float(info)], dtype=torch.float64, device="cuda"),
                    torch.tensor([anyd], dtype=torch.float64, device="cuda"), riw, m, sel)
        s = sel.cpu().numpy()
        status, eta, lsl, mult_ref = _host_rules(losses, etas, rr, info, anyd, riw, mult)
        assert int(s[2]) == status, (losses, rr, info, anyd, riw)
        assert float(m.item()) == mult_ref
        if status == 0:
            assert s[0] == eta and s[1] == lsl
    # theta update: accepted -> theta + eta delta (bit-identical to axpby), else theta
    th = torch.as_tensor(rng.normal(size=1001), device="cuda")
    d = torch.as_tensor(rng.normal(size=1001), device="cuda")
    d[5] = float("nan")
    out = torch.empty_like(th)
    K.theta_update(th, d, torch.tensor([0.25, 0, 1.0, 2], dtype=torch.float64, device="cuda"), out)
    assert torch.equal(out, th)  # rejected: untouched even where delta is NaN
    K.theta_update(th, d, torch.tensor([0.25, 0, 0.0, 2], dtype=torch.float64, device="cuda"), out)
    ref = K.axpby(0.25, d, 1.0, th)
    assert torch.equal(out.isnan(), ref.isnan())
    assert torch.equal(out[~out.isnan()], ref[~ref.isnan()])


CASES = [
    ("heat1d", {}, (2, 16, 16, 1), (60, 20, 20), 1e-3),           # J-free (factored Gram)
    ("poisson2d", {}, (2, 16, 16, 1), (60, 20), 1e-3),            # materialised J + SYRK
    ("allen_cahn", {}, (3, 16, 16, 1), (60, 20), 1e-3),           # embedding + cubic term
    ("poisson_ball_stde", dict(dim=10, index_set_size=3), (10, 16, 1), (40,), 1e3),
    ("poisson_ball_stde", dict(dim=200, index_set_size=4), (200, 16, 16, 1), (48,), 1e3),
    ("heat1d", {}, (2, 8, 1), (1, 1, 1), 1e-3),                  # m = 3
    ("poisson2d", {}, (2, 16, 1), (65, 64), 1e-3),               # ragged Cholesky blocks
]


def _run(P, monkeypatch, pname, kw, widths, counts, cap, pipelined, iters=6, **extra):
    if pipelined:
        monkeypatch.delenv("DNGD_NO_PIPELINE", raising=False)
    else:
        monkeypatch.setenv("DNGD_NO_PIPELINE", "1")
    config = P.OptimizerConfig(max_iters=iters, lam_cap=cap, deterministic_timing=True, **extra)
    return P.dngd_run(P.make_problem(pname, **kw), P.MlpSpec(widths), config, 5, counts=counts,
                      init="xavier_normal")


@pytest.mark.parametrize("pname,kw,widths,counts,cap", CASES)
def test_pipelined_loop_matches_eager(P, monkeypatch, pname, kw, widths, counts, cap):
    eager = _run(P, monkeypatch, pname, kw, widths, counts, cap, False)
    pipe = _run(P, monkeypatch, pname, kw, widths, counts, cap, True)
    assert not eager.aborted and not pipe.aborted
    assert len(eager.rows) == len(pipe.rows)
    for a, b in zip(eager.rows, pipe.rows):
        assert (a.iteration, a.wall_time) == (b.iteration, b.wall_time)
        np.testing.assert_array_equal([a.loss, a.lam, a.eta, a.ga_ratio, a.rel_l2],
                                      [b.loss, b.lam, b.eta, b.ga_ratio, b.rel_l2])
    assert np.array_equal(eager.final_theta.data, pipe.final_theta.data)


def test_pipelined_rollback_redoes_eagerly(P, monkeypatch):
    """A factorisation failure (status 2) or a non-finite loss (status 3) seen one
    step late: the queued successor is discarded, the iteration is redone on the
    host-driven path (retry ladder) and the pipeline resumes from its result.
    Simulated by reporting the status for iterations whose device step did not
    fail: the device state is put back to 'unchanged' as a real failure leaves it."""
    from paper_2505_21404_b200 import solver

    pname, kw, widths, counts, cap = CASES[0]
    eager = _run(P, monkeypatch, pname, kw, widths, counts, cap, False, iters=8)
    inputs = {}
    fake = {3: 2.0, 6: 3.0}  # fetch number -> reported status
    seen = {"n": 0}
    orig_enqueue = solver._DenseGraph.pipe_enqueue
    orig_fetch = solver._DenseGraph.pipe_fetch

    def enqueue(self, rmap):
        ticket = orig_enqueue(self, rmap)
        inputs[id(ticket[1])] = self.T[ticket[0]].clone()
        return ticket

    def fetch(self, ticket):
        arr, t_after, delta = orig_fetch(self, ticket)
        seen["n"] += 1
        if seen["n"] in fake:
            torch.cuda.synchronize()
            t_after.copy_(inputs[id(ticket[1])])  # what a failed step leaves behind
            arr = arr.copy()
            arr[6 + 31 + 2] = fake.pop(seen["n"])
        return arr, t_after, delta

    monkeypatch.setattr(solver._DenseGraph, "pipe_enqueue", enqueue)
    monkeypatch.setattr(solver._DenseGraph, "pipe_fetch", fetch)
    pipe = _run(P, monkeypatch, pname, kw, widths, counts, cap, True, iters=8)
    assert not fake
    assert not pipe.aborted
    assert len(pipe.rows) == len(eager.rows)
    np.testing.assert_allclose([r.loss for r in pipe.rows], [r.loss for r in eager.rows],
                               rtol=1e-9)
    assert [r.eta for r in pipe.rows][1:] == [r.eta for r in eager.rows][1:]
    np.testing.assert_allclose(pipe.final_theta.data, eager.final_theta.data, rtol=1e-8,
                               atol=1e-12)


def test_repeated_factorisation_failures_switch_to_ladder(P, monkeypatch):
    """Two consecutive iterations whose first factorisation fails: the pipelined
    loop stops paying a second Gram per iteration and finishes on the retry ladder
    applied to each iteration's own K; the trajectory is unchanged."""
    from paper_2505_21404_b200 import solver

    pname, kw, widths, counts, cap = CASES[0]
    eager = _run(P, monkeypatch, pname, kw, widths, counts, cap, False, iters=8)
    inputs = {}
    fake = {3: 2.0, 4: 2.0}
    seen = {"n": 0}
    orig_enqueue = solver._DenseGraph.pipe_enqueue
    orig_fetch = solver._DenseGraph.pipe_fetch

    def enqueue(self, rmap):
        ticket = orig_enqueue(self, rmap)
        inputs[id(ticket[1])] = self.T[ticket[0]].clone()
        return ticket

    def fetch(self, ticket):
        arr, t_after, delta = orig_fetch(self, ticket)
        seen["n"] += 1
        if seen["n"] in fake:
            torch.cuda.synchronize()
            t_after.copy_(inputs[id(ticket[1])])
            arr = arr.copy()
            arr[6 + 31 + 2] = fake.pop(seen["n"])
        return arr, t_after, delta

    monkeypatch.setattr(solver._DenseGraph, "pipe_enqueue", enqueue)
    monkeypatch.setattr(solver._DenseGraph, "pipe_fetch", fetch)
    pipe = _run(P, monkeypatch, pname, kw, widths, counts, cap, True, iters=8)
    assert not fake and not pipe.aborted
    assert len(pipe.rows) == len(eager.rows)
    np.testing.assert_allclose([r.loss for r in pipe.rows], [r.loss for r in eager.rows],
                               rtol=1e-9)
    assert [r.eta for r in pipe.rows][1:] == [r.eta for r in eager.rows][1:]
    assert [r.lam for r in pipe.rows][1:] == [r.lam for r in eager.rows][1:]
    from paper_2505_21404_b200._state import tls

    tls().graph_cache.clear()  # forget the learned ladder mode for later tests


def test_ladder_on_the_same_gram_matches_reference_ladder(P):
    """fused_dense_step(ladder=True) retries lam *= 10 on the K it formed; the damping
    it ends on and the step equal solver.dense_dual_solve's retry ladder
    (solver.py:161-173) at a lambda far below the conditioning floor."""
    from paper_2505_21404_b200.solver import fused_dense_step

    prob = P.make_problem("poisson2d")
    spec = P.MlpSpec((2, 32, 32, 1))
    colloc = prob.sample((300, 60), np.random.default_rng(2))
    rmap = P.PinnResidualMap(prob, spec, colloc)
    theta = P.xavier_normal_params(spec)
    for lam in (1e-16, 1e-13, 1e-3):
        step, losses, anyd, loss, r = fused_dense_step(rmap, theta, None, lam, True, 31,
                                                       ladder=True)
        _, g = rmap.residuals_and_gradient(theta)
        ref = P.dense_dual_solve(rmap, theta, g, lam=lam, use_ga=True)
        assert step.lambda_used == ref.lambda_used
        if lam >= 1e-3:  # (far below the floor the direction itself is not defined)
            d, e = step.delta.data, ref.delta.data
            assert np.linalg.norm(d - e) <= 1e-6 * np.linalg.norm(e)
    assert P.dense_dual_solve(rmap, theta, g, lam=1e-16, use_ga=False).lambda_used > 1e-16
