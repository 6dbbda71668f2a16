"""CPU (gloo, world_size 2) tests of the sharded step orchestration.

The per-rank numeric backend here is a small dense torch-CPU implementation
defined in this file (test infrastructure); what is under test is the product's
partitioning, collective sequence and replicated logic in
paper_2505_21404_b200/sharded.py -- the dense step, the Nystrom-PCG step and the
outer loop -- compared against the world_size-1 run.
"""

import os
import socket
import tempfile
from dataclasses import dataclass

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2505_21404_b200.sharded import (
    Comm,
    LocalComm,
    column_ranges,
    layer_row_ranges,
    row_ranges,
    sharded_dense_step,
    sharded_line_search,
    sharded_loop,
    sharded_pcg_step,
)


class DenseFactor:
    def __init__(self, K, lam):
        A = K + lam * torch.eye(K.shape[0], dtype=K.dtype)
        self.L, info = torch.linalg.cholesky_ex(A)
        self.ok = int(info) == 0

    def solve_(self, b):
        b.copy_(torch.cholesky_solve(b[:, None], self.L)[:, 0])
        return b


class FakeMap:
    """What the sharded outer loop reads from a residual map."""

    def __init__(self, r, J, Q):
        self.r, self.J, self.Q = r, J, Q
        self.m = r.shape[0]

    def residual(self, delta):
        return self.r + self.J @ delta + 0.5 * (self.Q @ (delta * delta))

    def loss(self, theta):
        rr = self.residual(theta.tensor - THETA0)
        return 0.5 * float(rr @ rr)

    def partition(self):
        return [("interior", 0, self.m)]


THETA0 = None


class TorchShardOps:
    """Dense stand-in for the CUDA ops: r(theta) = r0 + J d + Q (d*d)/2 with
    d = theta - theta0 (so J is the Jacobian and f_vv = Q (v*v) at theta0)."""

    def __init__(self, J, r, Q, rank, world, ranges):
        c0, c1 = ranges[rank]
        self.J, self.Jp, self.r, self.Q = J, J[:, c0:c1], r, Q
        self.rank = rank
        self.shard_sizes = [b - a for a, b in ranges]
        self.rows = row_ranges(J.shape[0], world)
        self.row_sizes = [b - a for a, b in self.rows]
        self.rmap = FakeMap(r, J, Q)
        self.theta = None

    def residuals(self):
        return self.r.clone()

    def gram_local(self):
        return self.Jp @ self.Jp.T

    def factor(self, K, lam):
        f = DenseFactor(K, lam)
        return f, f.ok

    def kmv(self, K, x, alpha):
        return alpha * (K @ x)

    def jt(self, y, scale):
        return scale * (self.Jp.T @ y)

    def jv(self, t_p):
        return self.Jp @ t_p

    def kcols(self, landmarks):
        return (self.Jp @ self.Jp[torch.as_tensor(landmarks)].T).contiguous()

    def dot(self, a, b):
        return (a * b).sum().reshape(1)

    def axpy(self, eta, delta, theta_t):
        return theta_t + eta * delta

    def fvv_rows(self, v):
        r0, r1 = self.rows[self.rank]
        return (self.Q @ (v * v))[r0:r1]

    def losses(self, theta, delta, etas):
        out = []
        for e in etas:
            rr = self.r + e * (self.J @ delta) + 0.5 * e * e * (self.Q @ (delta * delta))
            out.append(0.5 * float(rr @ rr))
        return torch.tensor(out, dtype=torch.float64)


class CpuNystrom:
    """solver.nystrom_from_columns restated in torch-CPU (the product's version
    runs its GEMMs in the CUDA library)."""

    def __init__(self, Kc, landmarks, lam):
        K_II = Kc[torch.as_tensor(landmarks)]
        K_II = 0.5 * (K_II + K_II.T)
        ev, Q = torch.linalg.eigh(K_II)
        keep = ev > 1e-10 * max(float(ev[-1]), 0.0)
        lam_q, Q = torch.flip(ev[keep], [0]), torch.flip(Q[:, keep], [1])
        Ut = Kc @ Q / lam_q
        Ut[torch.as_tensor(landmarks)] = Q
        U, S, _ = torch.linalg.svd(Ut * torch.sqrt(lam_q), full_matrices=False)
        self.U, self.lam_hat, self.lam = U, S * S, lam

    def apply_t(self, v):
        t = self.U.T @ v
        return self.U @ (t / (self.lam_hat + self.lam)) + (v - self.U @ t) / self.lam


def _problem(seed=0, m=23, n=57):
    g = torch.Generator().manual_seed(seed)
    J = torch.randn(m, n, generator=g, dtype=torch.float64)
    r = torch.randn(m, generator=g, dtype=torch.float64)
    Q = 0.01 * torch.randn(m, n, generator=g, dtype=torch.float64)
    return J, r, Q


def _run(comm, lam):
    J, r, Q = _problem()
    n = J.shape[1]
    ranges = column_ranges(n, comm.world)
    ops = TorchShardOps(J, r, Q, comm.rank, comm.world, ranges)
    res = sharded_dense_step(ops, comm, lam, use_ga=True)
    ls = sharded_line_search(ops, comm, None, res["delta"], 0.5 * float(r @ r))
    return res["delta"].numpy(), res["lambda_used"], res["ga_ratio"], ls.eta, ls.loss


def _run_pcg(comm, lam):
    J, r, Q = _problem(3, m=40, n=70)
    ranges = column_ranges(J.shape[1], comm.world)
    ops = TorchShardOps(J, r, Q, comm.rank, comm.world, ranges)
    res = sharded_pcg_step(ops, comm, lam, 12, 1e-10, 60, np.random.default_rng(7),
                           precond_factory=CpuNystrom)
    return res["delta"].numpy(), res["cg_iterations"]


@dataclass(frozen=True)
class _Cfg:
    lam_cap: float = 1e-2
    dense_threshold: int = 1000
    nystrom_rank: int = 8
    cg_tol: float = 1e-10
    cg_max_iters: int = 50
    use_ga: bool = True
    line_search_points: int = 31
    max_iters: int | None = 3
    wall_seconds: float | None = None
    resample: bool = True
    reject_if_worse: bool = False
    deterministic_timing: bool = True


def _run_loop(comm, pcg):
    """The sharded outer loop on a quadratic-in-delta map (Jacobian fixed at theta0)."""
    global THETA0
    from paper_2505_21404_b200.optimizer import TrainTrace
    from paper_2505_21404_b200.params import ParameterLayout, ParameterVector

    J, r, Q = _problem(5, m=30, n=44)
    THETA0 = torch.zeros(J.shape[1], dtype=torch.float64)
    ranges = column_ranges(J.shape[1], comm.world)
    layout = ParameterLayout([("theta", (J.shape[1],))])
    theta = ParameterVector(THETA0.clone(), layout)
    # PCG: a tolerance near the rounding floor, so the world-1 / world-2 iterates
    # differ by rounding rather than by where CG happened to stop
    cfg = _Cfg(dense_threshold=10, cg_tol=1e-14, cg_max_iters=200) if pcg else _Cfg()

    class LoopOps(TorchShardOps):
        """Residual / Jacobian re-linearised at the loop's current theta."""

        def residuals(self):
            d = self.theta.tensor - THETA0
            return self.rmap.residual(d)

        def losses(self, theta, delta, etas):
            d = theta.tensor - THETA0
            out = [0.5 * float(self.rmap.residual(d + e * delta) @ self.rmap.residual(d + e * delta))
                   for e in etas]
            return torch.tensor(out, dtype=torch.float64)

    def provider(it):
        return LoopOps(J, r, Q, comm.rank, comm.world, ranges)

    import paper_2505_21404_b200.sharded as S

    orig = S.sharded_pcg_step

    def pcg_cpu(ops, comm_, lam, ell, tol, iters, rng):
        return orig(ops, comm_, lam, ell, tol, iters, rng, precond_factory=CpuNystrom)

    S.sharded_pcg_step = pcg_cpu
    try:
        tr = sharded_loop(TrainTrace("quad", "dngd", 0), provider, theta, cfg, comm,
                          np.random.default_rng(1), "columns")
    finally:
        S.sharded_pcg_step = orig
    return ([row.loss for row in tr.rows], [row.eta for row in tr.rows],
            tr.final_theta.tensor.numpy(), tr.aborted)


def _worker(rank, world, port, out_path, lam):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        comm = Comm()
        delta, lam_used, ratio, eta, loss = _run(comm, lam)
        pd, pit = _run_pcg(comm, lam)
        ll, le, lt, la = _run_loop(comm, False)
        ql, qe, qt, qa = _run_loop(comm, True)
        if rank == 0:
            np.savez(out_path, delta=delta, lam_used=lam_used, ratio=ratio, eta=eta, loss=loss,
                     pcg_delta=pd, pcg_it=pit, loop_loss=ll, loop_eta=le, loop_theta=lt,
                     loop_abort=la, qloop_loss=ql, qloop_eta=qe, qloop_theta=qt, qloop_abort=qa)
    finally:
        dist.destroy_process_group()


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def test_column_ranges_cover_and_align():
    for n, w in [(12737, 2), (12737, 8), (1185, 4), (7, 8), (791553, 8)]:
        rg = column_ranges(n, w)
        assert rg[0][0] == 0 and rg[-1][1] == n
        assert all(a <= b for a, b in rg)
        assert all(rg[k][1] == rg[k + 1][0] for k in range(w - 1))
        assert all(a % 2 == 0 for a, _ in rg)


@pytest.mark.parametrize("widths", [(5, 512, 512, 512, 512, 1), (5, 1792, 1792, 1792, 1792, 1792, 1),
                                    (2, 64, 64, 64, 64, 1)])
@pytest.mark.parametrize("world", [1, 2, 4, 8])
def test_layer_row_ranges_on_gemm_rows(widths, world):
    """J-free shards: boundaries on layer starts or hidden-layer block rows, near-equal."""
    w = list(widths)
    L = len(w) - 1
    offs = np.cumsum([0] + [(w[k] + 1) * w[k + 1] for k in range(L)])
    n = int(offs[-1])
    rg = layer_row_ranges(widths, world)
    assert rg[0][0] == 0 and rg[-1][1] == n
    assert all(rg[k][1] == rg[k + 1][0] for k in range(world - 1))
    for b, _ in rg[1:]:
        k = int(np.searchsorted(offs, b, side="right")) - 1
        assert b == offs[k] or (1 <= k <= L - 2 and (b - offs[k]) % w[k + 1] == 0)
    sizes = [b - a for a, b in rg]
    if world > 1 and n > 100000:
        assert max(sizes) <= 1.02 * n / world  # balanced to within a GEMM row or two


@pytest.mark.parametrize("lam", [1e-3, 1e-1])
def test_sharded_step_world2_matches_world1(lam):
    ref = _run(LocalComm(), lam)
    # closed-form single-process check of the replicated algebra
    J, r, Q = _problem()
    K = J @ J.T
    A = K + lam * torch.eye(K.shape[0], dtype=torch.float64)
    y = torch.linalg.solve(A, -(K @ r))
    g = J.T @ r
    v = -(J.T @ y + g) / lam
    if ref[2] is not None and ref[2] > 0.5:  # GA gated off: delta is the GN direction
        assert np.allclose(ref[0], v.numpy(), rtol=1e-8, atol=1e-10)
    ref_pcg = _run_pcg(LocalComm(), lam)
    ref_loop = _run_loop(LocalComm(), False)
    ref_qloop = _run_loop(LocalComm(), True)
    # PCG at world 1 against the dense solve (tol 1e-10)
    Jp, rp, _ = _problem(3, m=40, n=70)
    Kp = Jp @ Jp.T
    yd = torch.linalg.solve(Kp + lam * torch.eye(40, dtype=torch.float64), -(Kp @ rp))
    dd = (-(Jp.T @ yd + Jp.T @ rp) / lam).numpy()
    assert np.linalg.norm(ref_pcg[0] - dd) <= 1e-5 * np.linalg.norm(dd)  # CG truncation at tol 1e-10
    with tempfile.TemporaryDirectory() as d:
        out = os.path.join(d, "res.npz")
        mp.spawn(_worker, args=(2, _free_port(), out, lam), nprocs=2, join=True)
        got = np.load(out)
    # K = K_0 + K_1 sums in a different order than J J^T: agreement at the
    # conditioning floor, not bitwise
    np.testing.assert_allclose(got["delta"], ref[0], rtol=1e-8, atol=1e-10)
    assert float(got["lam_used"]) == ref[1]
    assert abs(float(got["ratio"]) - ref[2]) <= 1e-8 * max(1.0, ref[2])
    assert float(got["eta"]) == ref[3]
    loss0 = 0.5 * float(r @ r)
    assert abs(float(got["loss"]) - ref[4]) <= 1e-10 * loss0
    # PCG: one m-vector all-reduce per product, Nystrom columns all-reduced
    assert abs(int(got["pcg_it"]) - ref_pcg[1]) <= 1
    # both stop at |r| <= 1e-10 |b|: each within its CG truncation of the dense answer
    assert np.linalg.norm(got["pcg_delta"] - dd) <= 1e-5 * np.linalg.norm(dd)
    assert np.linalg.norm(got["pcg_delta"] - ref_pcg[0]) <= 1e-5 * np.linalg.norm(dd)
    # the outer loop (dense and PCG dispatch): same rows and final theta
    for key, rl in (("loop", ref_loop), ("qloop", ref_qloop)):
        assert not bool(got[f"{key}_abort"]) and not rl[3]
        np.testing.assert_allclose(got[f"{key}_loss"], rl[0], rtol=1e-8, atol=1e-12 * rl[0][0])
        np.testing.assert_array_equal(got[f"{key}_eta"][1:], np.asarray(rl[1][1:]))
        np.testing.assert_allclose(got[f"{key}_theta"], rl[2], rtol=1e-7, atol=1e-9)
