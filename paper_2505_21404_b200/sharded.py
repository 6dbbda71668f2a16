"""The D-NGD step sharded across GPUs by parameter columns.

Rank p owns the contiguous parameter slice [c_p, c_{p+1}) of the reference layout
(model.py:48-54) and applies only its own J_p^T (north star: "each GPU applies its
own J_p^T alpha slice").  One dense step (solver.py:176-219) becomes

    r                                  replicated (every rank has every point)
    K   = sum_p K_p                    K_p local, one NCCL all-reduce (m x m)
    L   = chol(K + lam I)              replicated (identical K on every rank)
    y   = (K + lam I)^-1 (-K r)        replicated (b = -J g = -K r, g = J^T r)
    v_p = -J_p^T (y + r) / lam         local
    |v|^2                              all-reduce of one scalar
    v   = allgather(v_p)               n doubles, for f_vv
    f_vv rows of this rank's points    local, then allgather (m doubles)
    b_a = -K f_vv, y_a                 replicated
    a_p = -J_p^T (y_a + f_vv) / lam    local, |a|^2 all-reduced, GA gate
    delta = allgather(v_p + a_p/2)     for the line search
    line search                        candidates split across ranks, 31 losses gathered

Two per-rank backends (`ops`):
  * CudaShardOps  (configs 1, 2, 5): J_p materialised by the assembly kernel
    restricted to the rank's columns, K_p = J_p J_p^T on the FP64 tensor cores;
  * TileShardOps  (configs 3, 4, J-free): K_p = the rank's 1/P of the factored
    Gram's tiles, J_p^T w from the activations (dngd_jt_factored_range: only the
    rank's rows of each hidden-layer GEMM), shard boundaries on hidden-layer rows.
The forward/adjoint activation pass is replicated (every J_p row segment needs
every layer's adjoints); it is the Amdahl term.

The PCG step (solver.py:290-366) shards the same way: per CG iteration t_p =
J_p^T p local and ONE all-reduce of the m-vector J_p t_p; the Nystrom sketch
K[:, I] = sum_p J_p J_{I,p}^T is one all-reduce of m x ell; the preconditioner,
dots and CG control flow are replicated.

Collectives come from `Comm` (torch.distributed: NCCL on GPUs, gloo in the CPU
tests); the numeric operations from the rank's `ops` object.
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


def layer_row_ranges(widths, world: int) -> list[tuple[int, int]]:
    """Column shards for the J-free path: near-equal slices of [0, n) whose
    boundaries are layer starts or rows of a hidden layer's (w_k + 1) x w_{k+1}
    block, so every rank's J_p^T w is a set of whole GEMM rows."""
    if world < 1:
        raise ValueError("world must be >= 1")
    w = list(widths)
    L = len(w) - 1
    offs, off = [], 0
    for k in range(L):
        offs.append(off)
        off += (w[k] + 1) * w[k + 1]
    n = off
    cuts = {0, n}
    for k in range(L):
        cuts.add(offs[k])
        if 1 <= k <= L - 2:
            cuts.update(offs[k] + a * w[k + 1] for a in range(w[k] + 2))
    cuts = np.array(sorted(cuts))
    bounds = [0]
    for p in range(1, world):
        target = n * p / world
        j = int(np.argmin(np.abs(cuts - target)))
        bounds.append(max(bounds[-1], int(cuts[j])))
    bounds.append(n)
    return [(bounds[p], bounds[p + 1]) for p in range(world)]


def row_ranges(m: int, world: int) -> list[tuple[int, int]]:
    """Contiguous point rows per rank (f_vv and other per-point work)."""
    return column_ranges(m, world, align=1)


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
    y = y + r  # J^T (y + r) = J^T y + g
    v_p = ops.jt(y, -1.0 / lam_used)
    sizes = ops.shard_sizes
    vv = ops.dot(v_p, v_p)
    comm.allreduce_sum_(vv)
    v_norm = float(np.sqrt(_scalar(vv)))
    delta_p = v_p
    ga_ratio = None
    if use_ga and v_norm > GA_NORM_GUARD:
        v = comm.allgather_cat(v_p, sizes)
        f_vv = comm.allgather_cat(ops.fvv_rows(v), ops.row_sizes)
        y_a = ops.kmv(K, f_vv, -1.0)
        factor.solve_(y_a)
        y_a = y_a + f_vv
        a_p = ops.jt(y_a, -1.0 / lam_used)
        aa = ops.dot(a_p, a_p)
        comm.allreduce_sum_(aa)
        ga_ratio = 2.0 * float(np.sqrt(_scalar(aa))) / v_norm
        if ga_ratio <= GA_RATIO_MAX:
            delta_p = v_p + 0.5 * a_p
    delta = comm.allgather_cat(delta_p, sizes)
    return {"delta": delta, "lambda_used": lam_used, "ga_ratio": ga_ratio, "residuals": r,
            "cg_iterations": 0, "warning": None}


def sharded_pcg_step(ops, comm, lam: float, landmark_count: int, tol: float, max_iters: int,
                     rng, precond_factory=None) -> dict:
    """solver.py:290-366 with J column-sharded: b = -sum_p J_p g_p, the Nystrom
    columns sum_p J_p J_{I,p}^T and every CG product sum_p J_p (J_p^T p) are one
    all-reduce each; landmarks come from the run Generator on every rank (same
    draw everywhere); the final delta_p = -(J_p^T y + g_p)/lam is all-gathered."""
    from .solver import cg_iterate, nystrom_from_columns

    r = ops.residuals()
    g_p = ops.jt(r, 1.0)
    b = ops.jv(g_p)
    comm.allreduce_sum_(b)
    b.neg_()
    b_norm = float(b.norm().item())
    sizes = ops.shard_sizes
    if b_norm == 0.0:
        return {"delta": comm.allgather_cat(-(g_p / lam), sizes), "lambda_used": lam,
                "ga_ratio": None, "residuals": r, "cg_iterations": 0, "warning": None}
    m = r.shape[0]
    ell = int(landmark_count)
    landmarks = np.sort(rng.choice(m, size=ell, replace=False))
    Kc = ops.kcols(landmarks)
    comm.allreduce_sum_(Kc)
    precond = (precond_factory or nystrom_from_columns)(Kc, landmarks, lam)

    def apply_A(p):
        u = ops.jv(ops.jt(p, 1.0))
        comm.allreduce_sum_(u)
        return u.add_(p, alpha=lam)

    y, iterations, warning = cg_iterate(apply_A, precond, b, b_norm, tol, max_iters, ops.dot)
    delta_p = ops.jt(y + r, -1.0 / lam)  # -(J_p^T y + g_p)/lam
    return {"delta": comm.allgather_cat(delta_p, sizes), "lambda_used": lam, "ga_ratio": None,
            "residuals": r, "cg_iterations": iterations, "warning": warning}


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


# -- per-rank numeric backends on a B200 ---------------------------------------------------


class _CudaOpsBase:
    """What both backends share: replicated residuals, the factor, K x, dots,
    this rank's f_vv rows and line-search candidates."""

    def __init__(self, rmap, theta, ranges, rank, world):
        self.rmap = rmap
        self.theta = theta
        self.ranges = ranges
        self.rank, self.world = rank, world
        self.shard_sizes = [b - a for a, b in ranges]
        self.rows = row_ranges(rmap.m, world)
        self.row_sizes = [b - a for a, b in self.rows]

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

    def dot(self, a, b):
        from . import kernels as K

        return K.dot(a, b)

    def axpy(self, eta, delta, theta_t):
        """theta + eta delta (the same kernel as the single-GPU loop's update)."""
        from . import kernels as K

        return K.axpby(eta, delta, 1.0, theta_t)

    def fvv_rows(self, v):
        """f_vv of this rank's contiguous point rows (a sub-map of those points)."""
        import torch

        from .residuals import PinnResidualMap
        from .timing import stage

        r0, r1 = self.rows[self.rank]
        if r1 <= r0:
            return torch.zeros(0, dtype=torch.float64, device=v.device)
        if self.world == 1:
            return self.rmap.fvv_t(self.theta, v)
        colloc = self.rmap.collocation.subset(np.arange(r0, r1))
        sub = PinnResidualMap(self.rmap.problem, self.rmap.spec, colloc)
        with stage("fvv"):
            return sub.fvv_t(self.theta, v)

    def losses(self, theta, delta, etas):
        import torch

        if len(etas) == 0:
            return torch.zeros(0, dtype=torch.float64, device=delta.device)
        et = torch.as_tensor(np.ascontiguousarray(etas), device=delta.device)
        return self.rmap.losses_along_t(theta, delta, et)


class CudaShardOps(_CudaOpsBase):
    """Column shard with J_p materialised: rmap has col_range = ranges[rank]."""

    def __init__(self, rmap, theta, ranges, rank=None, world=None, pool=None):
        if rank is None:
            rank = next(i for i, rg in enumerate(ranges) if tuple(rg) == tuple(rmap.col_range))
        super().__init__(rmap, theta, ranges, rank, len(ranges) if world is None else world)
        self.pool = {} if pool is None else pool  # one J_p buffer shared by successive sets

    def _linearize(self):
        rm, pool = self.rmap, self.pool
        if rm._J is None and "J" in pool and pool["owner"] is not rm:
            pool["owner"]._cache = None  # its J contents are about to be overwritten
            rm._J = pool["J"]
        out = rm.linearize_t(self.theta)
        pool["J"], pool["owner"] = rm._J, rm
        return out

    def _J(self):
        return self._linearize()[1]

    def residuals(self):
        return self._linearize()[0]

    def gram_local(self):
        from . import kernels as K
        from .timing import stage

        with stage("syrk"):
            return K.syrk(self._J(), self.rmap.ncols)

    def jt(self, y, scale):
        from . import kernels as K

        with stage_("vjp"):
            return K.gemv_t(self._J(), y, self.rmap.ncols, None, scale)

    def jv(self, t_p):
        """J_p t_p (this rank's part of an m-vector that is all-reduced)."""
        from . import kernels as K

        with stage_("jvp"):
            return K.gemv_n(self._J(), t_p, self.rmap.ncols)

    def kcols(self, landmarks):
        """J_p J_{I,p}^T (m x ell), summed over the ranks by the caller."""
        import torch

        from . import kernels as K

        J = self._J()
        idx = torch.as_tensor(landmarks, device=J.device)
        with stage_("kcols"):
            return K.gemm_nt(J, J.index_select(0, idx), K=self.rmap.ncols).contiguous()


class TileShardOps(_CudaOpsBase):
    """J-free shard (configs 3-4): K_p = this rank's tiles of the factored Gram,
    J_p^T w from the activations; rmap is the full (col_range = all) map."""

    def residuals(self):
        return self.rmap.residuals_act_t(self.theta)

    def gram_local(self):
        import torch

        from . import kernels as K
        from .timing import stage

        rm = self.rmap
        d = rm._device()
        rm.residuals_act_t(self.theta)
        Kp = torch.zeros((rm.m, rm.m), dtype=torch.float64, device=d["device"])
        with stage("gram_kernel"):
            K.gram_factored_act(d["mlp"], d["arr"], d["nclass"], Kp, rm._act_workspace(),
                                self.rank, self.world)
        return Kp

    def jt(self, y, scale):
        import torch

        from . import kernels as K

        rm = self.rmap
        d = rm._device()
        rm.residuals_act_t(self.theta)  # activations of this theta (no-op when current)
        c0, c1 = self.ranges[self.rank]
        out = torch.empty(c1 - c0, dtype=torch.float64, device=d["device"])
        scratch = K.workspace("jt", K.jt_workspace_bytes(d["mlp"], d["arr"], d["nclass"]))
        with stage_("vjp"):
            K.jt_factored_range(d["mlp"], d["arr"], d["nclass"], y.contiguous(), scale, out,
                                c0, c1, rm._act_workspace(), scratch)
        return out


def stage_(name):
    from .timing import stage

    return stage(name)


# -- the sharded outer loop ------------------------------------------------------------------


def choose_layout(rmap, config) -> str:
    """'tiles' (J-free factored Gram, configs 3-4) or 'columns' (J_p materialised:
    narrow dense configs and Nystrom-PCG)."""
    if rmap.m < config.dense_threshold and rmap.jfree():
        return "tiles"
    return "columns"


def make_ops(layout, problem, spec, collocation, theta, comm, prev=None):
    """The rank's map and ops for one collocation set.  prev: the ops of an earlier
    set whose J_p buffer this one reuses (one m x n_p buffer per rank, not one per
    collocation set: 6.3 GB per rank at config 5, P = 8)."""
    from .residuals import PinnResidualMap

    if prev is not None and isinstance(prev, CudaShardOps):
        return CudaShardOps(PinnResidualMap(problem, spec, collocation, prev.rmap.col_range),
                            theta, prev.ranges, comm.rank, comm.world, prev.pool)
    n = spec.param_count()
    if layout == "tiles":
        ranges = layer_row_ranges(spec.layer_widths, comm.world)
        rmap = PinnResidualMap(problem, spec, collocation)
        return TileShardOps(rmap, theta, ranges, comm.rank, comm.world)
    ranges = column_ranges(n, comm.world)
    rmap = PinnResidualMap(problem, spec, collocation, col_range=ranges[comm.rank])
    return CudaShardOps(rmap, theta, ranges, comm.rank, comm.world)


def sharded_loop(trace, maps_provider, theta, config, comm, rng, layout, on_step=None,
                 rel_l2_fn=None):
    """optimizer._dngd_loop (optimizer.py:193-265) over the sharded step: the
    budget rule, damping with the rejection multiplier, the reject_if_worse test
    and the abort semantics of the reference loop.  maps_provider(iteration) ->
    ops for that iteration's collocation set (ops.theta is set here)."""
    from .optimizer import (LineSearchResult, StepResult, TraceRow, _Book, _budget_reached,
                            _Clock, lm_damping)
    from .params import ParameterVector

    clock = _Clock(config.deterministic_timing)
    ops = maps_provider(1)
    ops.theta = theta
    rel = rel_l2_fn(theta) if rel_l2_fn else float("nan")
    trace.rows.append(TraceRow(0, clock.stamp(), ops.rmap.loss(theta), rel_l2=rel))
    book = _Book(trace, config, clock, rel_l2_fn, on_step)
    book.rel_pending = None
    iteration = 0
    while True:
        iteration += 1
        if _budget_reached(config, iteration, clock):
            break
        try:
            ops = maps_provider(iteration)
            ops.theta = theta
            r = ops.residuals()
            loss = 0.5 * float(ops.dot(r, r).item())
            if not np.isfinite(loss):
                from .residuals import _raise_nonfinite

                _raise_nonfinite(r, ops.rmap.partition())
            lam = lm_damping(loss, config.lam_cap) * 10.0**book.rejections
            if ops.rmap.m < config.dense_threshold:
                res = sharded_dense_step(ops, comm, lam, config.use_ga)
            else:
                res = sharded_pcg_step(ops, comm, lam, min(config.nystrom_rank, ops.rmap.m),
                                       config.cg_tol, config.cg_max_iters, rng)
            step = StepResult(ParameterVector(res["delta"], theta.layout), res["lambda_used"],
                              res["cg_iterations"], ga_ratio=res["ga_ratio"],
                              warning=res["warning"])
            delta = res["delta"]
            if not bool(delta.any().item()):
                ls = LineSearchResult(1.0, loss, False, 0, False)
            else:
                with stage_("line_search_sharded"):
                    ls = sharded_line_search(ops, comm, theta, delta, loss,
                                             config.line_search_points)
        except Exception as exc:
            book.abort(iteration, exc)
            break
        if ls.rejected or (config.reject_if_worse and ls.loss > loss):
            if book.rejected(iteration, theta, step, ls, loss):
                break
            continue
        theta = ParameterVector(ops.axpy(ls.eta, delta, theta.tensor), theta.layout)
        book.accepted(iteration, theta, step, ls)
    trace.final_theta = theta
    return trace


def sharded_dngd_run(problem, spec, config, seed: int, comm=None, counts=None,
                     init: str = "xavier_normal", on_step=None, layout: str = "auto",
                     track_rel_l2: bool = False):
    """dngd_run (optimizer.py:290-314) with the column-sharded step.

    Every rank draws the same collocation points and landmarks (same seed, same
    Generator call order), so residuals, K and the replicated solves agree
    across ranks; each rank applies only its own J_p^T.  layout: 'tiles'
    (J-free, configs 3-4), 'columns' (J_p materialised: configs 1-2 and the
    Nystrom-PCG config 5) or 'auto'."""
    from dataclasses import replace

    from .model import INITIALIZERS
    from .optimizer import TrainTrace, _rel_l2_fn
    from .problems import sample_collocation
    from .residuals import PinnResidualMap

    comm = comm or Comm()
    spec = replace(spec, seed=seed)
    rng = np.random.default_rng(seed)
    theta = INITIALIZERS[init](spec)
    state = {"colloc": None, "ops": None}
    if layout == "auto":
        probe = PinnResidualMap(problem, spec, sample_collocation(problem, counts,
                                                                   np.random.default_rng(seed)))
        layout = choose_layout(probe, config)

    def provider(iteration):
        if state["colloc"] is None or (config.resample and iteration > 1):
            state["colloc"] = sample_collocation(problem, counts, rng)
            state["ops"] = make_ops(layout, problem, spec, state["colloc"], theta, comm,
                                    prev=state["ops"])
        return state["ops"]

    trace = TrainTrace(problem=problem.name, method=f"dngd-sharded-{layout}", seed=seed)
    rel_fn = _rel_l2_fn(problem, spec) if track_rel_l2 else None
    return sharded_loop(trace, provider, theta, config, comm, rng, layout, on_step, rel_fn)
