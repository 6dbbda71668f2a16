"""CPU (gloo, world_size 2) test of the column-sharded step orchestration.

The per-rank numeric backend here is a small dense torch-CPU implementation
defined in this file (test infrastructure); what is under test is the product's
partitioning, collective sequence and replicated logic in
paper_2505_21404_b200/sharded.py, compared against the world_size-1 run.
"""

import os
import socket
import tempfile

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2505_21404_b200.sharded import (
    Comm,
    LocalComm,
    column_ranges,
    sharded_dense_step,
    sharded_line_search,
)


class DenseFactor:
    def __init__(self, K, lam):
        A = K + lam * torch.eye(K.shape[0], dtype=K.dtype)
        self.L, info = torch.linalg.cholesky_ex(A)
        self.ok = int(info) == 0

    def solve_(self, b):
        b.copy_(torch.cholesky_solve(b[:, None], self.L)[:, 0])
        return b


class TorchShardOps:
    """Dense stand-in for CudaShardOps: J given explicitly, f_vv and losses closed form."""

    def __init__(self, J, r, Q, rank, ranges):
        c0, c1 = ranges[rank]
        self.J, self.Jp, self.r, self.Q = J, J[:, c0:c1], r, Q
        self.shard_sizes = [b - a for a, b in ranges]

    def residuals(self):
        return self.r.clone()

    def grad_local(self, r):
        return self.Jp.T @ r

    def gram_local(self):
        return self.Jp @ self.Jp.T

    def factor(self, K, lam):
        f = DenseFactor(K, lam)
        return f, f.ok

    def kmv(self, K, x, alpha):
        return alpha * (K @ x)

    def jt(self, y, g, scale):
        out = self.Jp.T @ y
        return scale * (out + g) if g is not None else scale * out

    def dot(self, a, b):
        return (a * b).sum()

    def fvv(self, v):  # a curved map: f_vv = Q (v*v)
        return self.Q @ (v * v)

    def losses(self, theta, delta, etas):
        out = []
        for e in etas:
            rr = self.r + e * (self.J @ delta) + 0.5 * e * e * (self.Q @ (delta * delta))
            out.append(0.5 * float(rr @ rr))
        return torch.tensor(out, dtype=torch.float64)


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
    ops = TorchShardOps(J, r, Q, comm.rank, ranges)
    res = sharded_dense_step(ops, comm, lam, use_ga=True)
    ls = sharded_line_search(ops, comm, None, res["delta"], 0.5 * float(r @ r))
    return res["delta"].numpy(), res["lambda_used"], res["ga_ratio"], ls.eta, ls.loss


def _worker(rank, world, port, out_path, lam):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        delta, lam_used, ratio, eta, loss = _run(Comm(), lam)
        if rank == 0:
            np.savez(out_path, delta=delta, lam_used=lam_used, ratio=ratio, eta=eta, loss=loss)
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
