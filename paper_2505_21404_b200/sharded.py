"""Column-sharded D-NGD step across GPUs.

Rank p owns the contiguous parameter slice [c_p, c_{p+1}) of the reference
layout (model.py:48-54) and materialises only J_p = J[:, c_p:c_{p+1}].  One dense
step (solver.py:176-219) becomes

    K_p = J_p J_p^T                    local FP64 tensor-core SYRK
    K   = sum_p K_p                    ncclAllReduce over NVLink (m x m)
    L   = chol(K + lam I)              replicated (identical K on every rank)
    b   = -K r  (= -J g, g = J^T r)    replicated, no communication
    v_p = -(J_p^T y + g_p) / lam       local
    |v|^2                              all-reduce of one scalar
    v   = allgather(v_p)               n doubles, for f_vv
    f_vv, b_a = -K f_vv, y_a           replicated
    a_p = -J_p^T (y_a + f_vv) / lam    local, |a|^2 all-reduced
    delta = allgather(v_p + a_p/2)     for the line search
    line search                        candidates split across ranks, 31 losses gathered

The residuals r and the forward/adjoint activations are computed redundantly on
every rank (the J_p row segments need every layer's adjoints).  The numeric
operations come from a per-rank `ops` object (CudaShardOps on B200 ranks); the
collectives from `Comm` (torch.distributed: NCCL on GPUs, gloo in the CPU tests).
"""

from __future__ import annotations

import numpy as np

from .errors import FactorizationError
from .solver import GA_NORM_GUARD, GA_RATIO_MAX


def column_ranges(n: int, world: int, align: int = 2) -> list[tuple[int, int]]:
    """Split [0, n) into `world` contiguous ranges of near-equal size with
    boundaries on multiples of `align` (16-byte aligned J_p row starts)."""
    if world < 1:
        raise ValueError("world must be >= 1")
    bounds = [0]
    for p in range(1, world):
        b = int(round(n * p / world))
        b -= b % align
        bounds.append(max(bounds[-1], min(b, n)))
    bounds.append(n)
    return [(bounds[p], bounds[p + 1]) for p in range(world)]


class Comm:
    """The collectives of the sharded step over torch.distributed."""

    def __init__(self, group=None):
        import torch.distributed as dist

        self.dist = dist
        self.group = group
        self.rank = dist.get_rank(group)
        self.world = dist.get_world_size(group)

    def allreduce_sum_(self, t):
        if self.world > 1:
            self.dist.all_reduce(t, op=self.dist.ReduceOp.SUM, group=self.group)
        return t

    def allgather_cat(self, t_local, sizes):
        """Concatenate per-rank 1-d tensors of (possibly unequal) `sizes`."""
        import torch

        if self.world == 1:
            return t_local
        mx = max(sizes)
        buf = torch.zeros(mx, dtype=t_local.dtype, device=t_local.device)
        buf[: t_local.numel()] = t_local
        out = torch.empty(self.world * mx, dtype=t_local.dtype, device=t_local.device)
        self.dist.all_gather_into_tensor(out, buf, group=self.group)
        return torch.cat([out[p * mx : p * mx + sizes[p]] for p in range(self.world)])


class LocalComm:
    """world = 1 stand-in (single process, no collectives)."""

    rank = 0
    world = 1

    def allreduce_sum_(self, t):
        return t

    def allgather_cat(self, t_local, sizes):
        return t_local


def _scalar(x) -> float:
    return float(x.item()) if hasattr(x, "item") else float(x)


def sharded_dense_step(ops, comm, lam: float, use_ga: bool = True, retries: int = 5) -> dict:
    """One column-sharded dense dual step; returns the full (replicated) step."""
    r = ops.residuals()
    g_p = ops.grad_local(r)
    K = ops.gram_local()
    comm.allreduce_sum_(K)
    lam_used = lam
    factor = None
    for _ in range(retries + 1):
        factor, ok = ops.factor(K, lam_used)
        if ok:
            break
        lam_used *= 10.0
    else:
        raise FactorizationError(
            f"Cholesky of the damped Gramian failed after {retries} retries "
            f"(final damping {lam_used:.3e})"
        )
    y = ops.kmv(K, r, -1.0)  # b = -K r = -J g
    factor.solve_(y)
    v_p = ops.jt(y, g_p, -1.0 / lam_used)
    sizes = ops.shard_sizes
    vv = ops.dot(v_p, v_p)
    comm.allreduce_sum_(vv)
    v_norm = float(np.sqrt(_scalar(vv)))
    delta_p = v_p
    ga_ratio = None
    if use_ga and v_norm > GA_NORM_GUARD:
        v = comm.allgather_cat(v_p, sizes)
        f_vv = ops.fvv(v)
        y_a = ops.kmv(K, f_vv, -1.0)
        factor.solve_(y_a)
        y_a = y_a + f_vv
        a_p = ops.jt(y_a, None, -1.0 / lam_used)
        aa = ops.dot(a_p, a_p)
        comm.allreduce_sum_(aa)
        ga_ratio = 2.0 * float(np.sqrt(_scalar(aa))) / v_norm
        if ga_ratio <= GA_RATIO_MAX:
            delta_p = v_p + 0.5 * a_p
    delta = comm.allgather_cat(delta_p, sizes)
    return {"delta": delta, "lambda_used": lam_used, "ga_ratio": ga_ratio, "residuals": r}


def sharded_line_search(ops, comm, theta, delta, current_loss, points_count: int = 31):
    """optimizer.py:148-166 with the candidates split across ranks (contiguous
    blocks) and the losses gathered; identical selection rule."""
    import torch

    from .optimizer import _select

    etas = 2.0 ** -np.arange(points_count, dtype=np.float64)
    blocks = column_ranges(points_count, comm.world, align=1)
    lo, hi = blocks[comm.rank]
    local = ops.losses(theta, delta, etas[lo:hi])
    sizes = [b - a for a, b in blocks]
    if not torch.is_tensor(local):
        local = torch.as_tensor(local)
    losses = comm.allgather_cat(local, sizes)
    return _select(losses.cpu().numpy(), etas, current_loss, points_count)


class CudaShardOps:
    """Per-rank numeric operations on a B200 for one collocation set and θ."""

    def __init__(self, rmap, theta, ranges):
        self.rmap = rmap  # PinnResidualMap with col_range = ranges[rank]
        self.theta = theta
        self.shard_sizes = [b - a for a, b in ranges]

    def residuals(self):
        r, _ = self.rmap.linearize_t(self.theta)
        return r

    def grad_local(self, r):
        from . import kernels as K

        _, J = self.rmap.linearize_t(self.theta)
        return K.gemv_t(J, r, self.rmap.ncols)

    def gram_local(self):
        from . import kernels as K
        from .timing import stage

        _, J = self.rmap.linearize_t(self.theta)
        with stage("syrk"):
            return K.syrk(J, self.rmap.ncols)

    def factor(self, K, lam):
        from .solver import _Factor
        from .timing import stage

        fac = _Factor.get(K.shape[0], K.device)
        with stage("potrf"):
            fac.factor(K, lam)
        return fac, int(fac.info.item()) == 0

    def kmv(self, K, x, alpha):
        from . import kernels as Kn

        return Kn.gemv_n(K, x, alpha=alpha)

    def jt(self, y, g, scale):
        from . import kernels as K

        _, J = self.rmap.linearize_t(self.theta)
        return K.gemv_t(J, y, self.rmap.ncols, g, scale)

    def dot(self, a, b):
        from . import kernels as K

        return K.dot(a, b)

    def fvv(self, v):
        return self.rmap.fvv_t(self.theta, v)

    def losses(self, theta, delta, etas):
        import torch

        if len(etas) == 0:
            return torch.zeros(0, dtype=torch.float64, device=delta.device)
        et = torch.as_tensor(np.ascontiguousarray(etas), device=delta.device)
        return self.rmap.losses_along_t(theta, delta, et)


def sharded_dngd_run(problem, spec, config, seed: int, comm=None, counts=None,
                     init: str = "xavier_normal", on_step=None):
    """dngd_run (optimizer.py:290-314) with the column-sharded dense step.

    Every rank draws the same collocation points (same seed, same Generator call
    order), so residuals, K and the replicated solves agree across ranks; each
    rank assembles only its own Jacobian columns.  Dense dispatch only (PCG
    sharding is not part of this build)."""
    from dataclasses import replace

    import torch

    from . import kernels as K
    from .model import INITIALIZERS
    from .optimizer import (MAX_CONSECUTIVE_REJECTIONS, LineSearchResult, TraceRow,
                            TrainTrace, _Clock, lm_damping)
    from .params import ParameterVector
    from .problems import sample_collocation
    from .residuals import PinnResidualMap

    comm = comm or Comm()
    spec = replace(spec, seed=seed)
    rng = np.random.default_rng(seed)
    theta = INITIALIZERS[init](spec)
    ranges = column_ranges(spec.param_count(), comm.world)
    clock = _Clock(config.deterministic_timing)
    trace = TrainTrace(problem=problem.name, method="dngd-sharded", seed=seed)
    rmap = PinnResidualMap(problem, spec, sample_collocation(problem, counts, rng),
                           col_range=ranges[comm.rank])
    if rmap.m >= config.dense_threshold:
        raise NotImplementedError("the sharded step covers the dense dispatch only")
    trace.rows.append(TraceRow(0, clock.stamp(), rmap.loss(theta)))
    rejections = 0
    for iteration in range(1, (config.max_iters or 0) + 1):
        if config.resample and iteration > 1:
            rmap = rmap.rebind(sample_collocation(problem, counts, rng))
        ops = CudaShardOps(rmap, theta, ranges)
        r = ops.residuals()
        loss = 0.5 * float(K.dot(r, r).item())
        lam = lm_damping(loss, config.lam_cap) * 10.0**rejections
        try:
            step = sharded_dense_step(ops, comm, lam, config.use_ga)
        except Exception as exc:
            trace.aborted = True
            trace.abort_reason = f"error at iteration {iteration}: {exc!r}"
            break
        delta = step["delta"]
        if not bool(delta.any().item()):
            ls = LineSearchResult(1.0, loss, False, 0, False)
        else:
            ls = sharded_line_search(ops, comm, theta, delta, loss, config.line_search_points)
        if ls.rejected:
            rejections += 1
            trace.rows.append(TraceRow(iteration, clock.stamp(), loss, lam=step["lambda_used"]))
            if on_step is not None:
                on_step(iteration, theta, step, ls)
            if rejections >= MAX_CONSECUTIVE_REJECTIONS:
                trace.aborted = True
                trace.abort_reason = f"{rejections} consecutive step rejections"
                break
            continue
        rejections = 0
        theta = ParameterVector(K.axpby(ls.eta, delta, 1.0, theta.tensor), theta.layout)
        if on_step is not None:
            on_step(iteration, theta, step, ls)
        ga = step["ga_ratio"]
        trace.rows.append(TraceRow(iteration, clock.stamp(), ls.loss, lam=step["lambda_used"],
                                   eta=ls.eta, ga_ratio=ga if ga is not None else float("nan")))
    trace.final_theta = theta
    return trace
