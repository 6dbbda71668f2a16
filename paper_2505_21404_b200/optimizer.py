"""Outer D-NGD loop on the GPU backend (reference optimizer.py:1-314).

Same configuration schema (OptimizerConfig fields and validation), damping
rule, line-search semantics, rejection ladder, trace rows and seeding
discipline as the reference, so traces are row-for-row comparable.  The
parameters, residuals, Jacobian and all step algebra stay on the device; per
iteration the host sees a handful of scalars (loss, lambda, 31 line-search
losses, GA ratio) and the freshly sampled collocation points it uploads.
"""

from __future__ import annotations

import time
from dataclasses import dataclass, field, replace

import numpy as np

from .errors import ConfigError, DomainError
from .model import INITIALIZERS, MlpSpec
from .params import ParameterVector
from .residuals import PinnResidualMap, ResidualMap
from .solver import StepResult, dense_dual_solve, dense_iteration, fused_dense_step, pcg_step
from .timing import stage

LAMBDA_FLOOR = 1e-12
MAX_CONSECUTIVE_REJECTIONS = 10


@dataclass(frozen=True)
class OptimizerConfig:
    """Knobs of the outer loop; exactly one budget kind must be set (optimizer.py:26-71)."""

    lam_cap: float = 1e-5
    dense_threshold: int = 4000
    nystrom_rank: int = 64
    cg_tol: float = 1e-10
    cg_max_iters: int = 500
    use_ga: bool = True
    line_search_points: int = 31
    max_iters: int | None = None
    wall_seconds: float | None = None
    resample: bool = True
    reject_if_worse: bool = False
    deterministic_timing: bool = False

    def __post_init__(self):
        if self.lam_cap <= 0.0:
            raise ConfigError(f"lam_cap must be positive, got {self.lam_cap}", "lam_cap")
        if self.line_search_points < 1:
            raise ConfigError(
                f"line_search_points must be >= 1, got {self.line_search_points}",
                "line_search_points",
            )
        if self.dense_threshold < 1:
            raise ConfigError(
                f"dense_threshold must be >= 1, got {self.dense_threshold}", "dense_threshold"
            )
        if self.nystrom_rank < 1:
            raise ConfigError(f"nystrom_rank must be >= 1, got {self.nystrom_rank}", "nystrom_rank")
        if self.cg_tol <= 0.0 or self.cg_max_iters < 1:
            raise ConfigError("CG tolerance and iteration cap must be positive", "cg_tol")
        if (self.max_iters is None) == (self.wall_seconds is None):
            raise ConfigError("exactly one of max_iters / wall_seconds must be set", "max_iters")
        if self.max_iters is not None and self.max_iters < 1:
            raise ConfigError(f"max_iters must be >= 1, got {self.max_iters}", "max_iters")
        if self.wall_seconds is not None and self.wall_seconds <= 0.0:
            raise ConfigError(
                f"wall_seconds must be positive, got {self.wall_seconds}", "wall_seconds"
            )


@dataclass
class TraceRow:
    iteration: int
    wall_time: float
    loss: float
    rel_l2: float = float("nan")
    lam: float = float("nan")
    eta: float = float("nan")
    cg_iterations: int = 0
    ga_ratio: float = float("nan")


@dataclass
class TrainTrace:
    problem: str
    method: str
    seed: int
    rows: list[TraceRow] = field(default_factory=list)
    final_theta: ParameterVector | None = None
    aborted: bool = False
    abort_reason: str | None = None
    abort_traceback: str | None = None  # not in the reference trace schema (diagnostics)
    diverged: bool = False

    @property
    def final_loss(self) -> float:
        return self.rows[-1].loss if self.rows else float("nan")

    @property
    def final_rel_l2(self) -> float:
        return self.rows[-1].rel_l2 if self.rows else float("nan")


class _Clock:
    """Strictly increasing stamps; logical ticks in deterministic mode (optimizer.py:110-129)."""

    def __init__(self, deterministic: bool):
        self.deterministic = deterministic
        self.t0 = time.monotonic()
        self.ticks = 0
        self.last = 0.0

    def stamp(self) -> float:
        self.ticks += 1
        if self.deterministic:
            t = float(self.ticks)
        else:
            t = max(time.monotonic() - self.t0, self.last + 1e-9)
        self.last = t
        return t

    def elapsed(self) -> float:
        return time.monotonic() - self.t0


def lm_damping(loss: float, lam_cap: float) -> float:
    """optimizer.py:132-136."""
    if loss < 0.0:
        raise DomainError(f"loss must be nonnegative, got {loss}")
    return max(min(loss, lam_cap), LAMBDA_FLOOR)


@dataclass
class LineSearchResult:
    eta: float | None
    loss: float
    degraded: bool
    evaluations: int
    rejected: bool


def _select(losses: np.ndarray, etas: np.ndarray, current_loss, points_count) -> LineSearchResult:
    finite = np.isfinite(losses)
    if not finite.any():
        return LineSearchResult(None, float("nan"), False, points_count, True)
    j = int(np.argmin(np.where(finite, losses, np.inf)))
    degraded = current_loss is not None and losses[j] > current_loss
    return LineSearchResult(float(etas[j]), float(losses[j]), degraded, points_count, False)


def line_search(loss_many, theta, delta, current_loss: float | None = None,
                points_count: int = 31) -> LineSearchResult:
    """Grid search over eta = 2^0 ... 2^-(count-1) (optimizer.py:148-166)."""
    theta = np.asarray(theta, dtype=np.float64)
    delta = np.asarray(delta, dtype=np.float64)
    etas = 2.0 ** -np.arange(points_count, dtype=np.float64)
    candidates = theta[None, :] + etas[:, None] * delta[None, :]
    losses = np.asarray(loss_many(candidates), dtype=np.float64)
    return _select(losses, etas, current_loss, points_count)


def device_line_search(rmap: ResidualMap, theta: ParameterVector, delta_t,
                       current_loss: float | None, points_count: int = 31) -> LineSearchResult:
    """line_search with the candidate losses evaluated by the batched device kernel;
    identical selection rule (ties -> larger eta, non-finite skipped, all non-finite
    -> rejected)."""
    import torch

    key = (points_count, str(delta_t.device))
    from ._state import tls

    etas_tab = tls().etas
    etas_t = etas_tab.get(key)
    if etas_t is None:
        etas_t = etas_tab[key] = torch.as_tensor(
            2.0 ** -np.arange(points_count, dtype=np.float64), device=delta_t.device
        )
    losses = rmap.losses_along_t(theta, delta_t, etas_t).cpu().numpy()
    return _select(losses, etas_t.cpu().numpy(), current_loss, points_count)


# -- the main loop ------------------------------------------------------------------------


def _dispatch_step(rmap: ResidualMap, theta, g, lam: float, config: OptimizerConfig,
                   rng) -> StepResult:
    """optimizer.py:172-184."""
    if rmap.m < config.dense_threshold:
        return dense_dual_solve(rmap, theta, g, lam=lam, use_ga=config.use_ga)
    return pcg_step(
        rmap,
        theta,
        g,
        lam=lam,
        landmark_count=min(config.nystrom_rank, rmap.m),
        tol=config.cg_tol,
        max_iters=config.cg_max_iters,
        rng=rng,
    )


def _budget_reached(config: OptimizerConfig, iteration: int, clock: _Clock) -> bool:
    if config.max_iters is not None:
        return iteration > config.max_iters
    return clock.elapsed() >= config.wall_seconds


def _eager_body(rmap, theta, config: OptimizerConfig, rng, rejections: int, redo=False):
    """One iteration up to the line-search result (optimizer.py:216-229): returns
    (step, ls, loss).  redo=True skips the fused device attempt (known to fail its
    factorisation) and goes straight to the retry ladder."""
    from . import kernels as K

    fused = None
    dense = rmap.m < config.dense_threshold
    jfree = dense and getattr(rmap, "jfree", lambda: False)()
    mult = 10.0**rejections
    if dense and not redo:
        # device-resident damping, step and line search: one host sync
        # (solver.fused_dense_step); loss comes back with the losses
        fused = dense_iteration(rmap, theta, config.use_ga, config.line_search_points,
                                config.lam_cap, mult)
        loss, r = fused[3], fused[4]
        J = None
        if fused[0] is None:
            fused = None  # factorisation failed: eager path keeps the retry ladder
            J = None if jfree else rmap.jacobian_t(theta)  # only the fallback needs J
    elif dense and isinstance(rmap, PinnResidualMap):
        # the retry ladder on the K this iteration forms (solver.fused_dense_step
        # with ladder=True): a failed factorisation costs one potrf, not a new Gram
        from .solver import fused_dense_step

        fused = fused_dense_step(rmap, theta, None, None, config.use_ga,
                                 config.line_search_points, lam_cap=config.lam_cap,
                                 lam_mult=mult, ladder=True)
        loss, r = fused[3], fused[4]
        J = None
    elif dense:
        if jfree:
            r, J = rmap.residuals_act_t(theta), None
        else:
            r, J = rmap.linearize_t(theta)
        loss = 0.5 * float(K.dot(r, r).item())
    else:
        jfree = bool(getattr(rmap, "jfree_pcg", lambda: False)())
        if jfree:  # J-free PCG: residuals and activations only
            r, J = rmap.residuals_act_t(theta), None
        else:
            r, J = rmap.linearize_t(theta)
        loss = 0.5 * float(K.dot(r, r).item())
    if not np.isfinite(loss):
        from .residuals import _raise_nonfinite

        _raise_nonfinite(r, rmap.partition())
    lam = lm_damping(loss, config.lam_cap) * mult
    if fused is None:
        g = None
        if not jfree:
            with stage("gemv"):
                g = K.gemv_t(J, r, rmap.n)
        step = _dispatch_step(rmap, theta, g, lam, config, rng)
    else:
        step = fused[0]
    delta_t = step.delta.tensor
    if fused is not None:
        etas = 2.0 ** -np.arange(config.line_search_points, dtype=np.float64)
        if not fused[2]:
            ls = LineSearchResult(1.0, loss, False, 0, False)
        else:
            ls = _select(fused[1], etas, loss, config.line_search_points)
    elif not bool(delta_t.any().item()):
        ls = LineSearchResult(1.0, loss, False, 0, False)
    else:
        ls = device_line_search(rmap, theta, delta_t, loss, config.line_search_points)
    return step, ls, loss


class _Book:
    """Row bookkeeping shared by the eager and the pipelined loop (optimizer.py:226-262)."""

    def __init__(self, trace, config, clock, rel_l2_fn, on_step):
        self.trace, self.config, self.clock = trace, config, clock
        self.rel_l2_fn, self.on_step = rel_l2_fn, on_step
        self.rejections = 0
        self.rel_pending = []  # (row, handle) of asynchronous rel-L2 evaluations
        self.snapshot = False  # on_step gets a copy (theta lives in a reused buffer)

    def _user_theta(self, theta):
        # callbacks that only count iterations can opt out: fn.needs_theta = False
        if self.snapshot and getattr(self.on_step, "needs_theta", True):
            return ParameterVector(theta.tensor.clone(), theta.layout)
        return theta

    def _rel(self, theta, row):
        fn = self.rel_l2_fn
        if fn is None:
            return
        if getattr(fn, "enqueue", None) is not None and self.rel_pending is not None:
            self.rel_pending.append((row, fn.enqueue(theta)))
        else:
            row.rel_l2 = fn(theta)

    def resolve(self, keep: int = 0):
        """Fill the rel-L2 of all but the last `keep` pending rows."""
        fn = self.rel_l2_fn
        while len(self.rel_pending) > keep:
            row, h = self.rel_pending.pop(0)
            row.rel_l2 = fn.fetch(h)

    def rejected(self, iteration, theta, step, ls, loss) -> bool:
        """Record a rejected step; True when the loop must stop."""
        self.rejections += 1
        row = TraceRow(iteration, self.clock.stamp(), loss, lam=step.lambda_used,
                       cg_iterations=step.cg_iterations)
        self._rel(theta, row)
        self.trace.rows.append(row)
        if self.on_step is not None:
            self.on_step(iteration, self._user_theta(theta), step, ls)
        if self.rejections >= MAX_CONSECUTIVE_REJECTIONS:
            self.trace.aborted = True
            self.trace.abort_reason = (
                f"{self.rejections} consecutive step rejections; last damping "
                f"{step.lambda_used:.3e}"
            )
            return True
        return False

    def accepted(self, iteration, theta_new, step, ls):
        self.rejections = 0
        if self.on_step is not None:
            self.on_step(iteration, self._user_theta(theta_new), step, ls)
        row = TraceRow(iteration, self.clock.stamp(), ls.loss, lam=step.lambda_used, eta=ls.eta,
                       cg_iterations=step.cg_iterations,
                       ga_ratio=step.ga_ratio if step.ga_ratio is not None else float("nan"))
        self._rel(theta_new, row)
        self.trace.rows.append(row)

    def abort(self, iteration, exc):
        import traceback

        self.trace.aborted = True
        self.trace.abort_reason = f"error at iteration {iteration}: {exc!r}"
        self.trace.abort_traceback = "".join(traceback.format_exception(exc))


def _pipeline_ok(rmap, config) -> bool:
    import os

    from .solver import graph_eligible

    return (os.environ.get("DNGD_NO_PIPELINE") is None and rmap.m < config.dense_threshold
            and isinstance(rmap, PinnResidualMap) and graph_eligible(rmap))


def _dngd_loop(trace: TrainTrace, rmap_provider, theta: ParameterVector, config: OptimizerConfig,
               rng, rel_l2_fn=None, on_step=None) -> TrainTrace:
    """optimizer.py:193-265 with device-resident state.  Dense PINN iterations run
    pipelined (_pipelined_loop); everything else step by step."""
    from . import kernels as K

    clock = _Clock(config.deterministic_timing)
    rmap = rmap_provider(1)
    rel = rel_l2_fn(theta) if rel_l2_fn else float("nan")
    trace.rows.append(TraceRow(0, clock.stamp(), rmap.loss(theta), rel_l2=rel))
    book = _Book(trace, config, clock, rel_l2_fn, on_step)
    if _pipeline_ok(rmap, config):
        theta = _pipelined_loop(book, rmap_provider, theta, config, rng)
        trace.final_theta = theta
        return trace
    book.rel_pending = None  # eager loop: rel-L2 evaluated in place
    iteration = 0
    while True:
        iteration += 1
        if _budget_reached(config, iteration, clock):
            break
        try:
            rmap = rmap_provider(iteration)
            step, ls, loss = _eager_body(rmap, theta, config, rng, book.rejections)
        except Exception as exc:
            book.abort(iteration, exc)
            break
        if ls.rejected or (config.reject_if_worse and ls.loss > loss):
            if book.rejected(iteration, theta, step, ls, loss):
                break
            continue
        theta = ParameterVector(K.axpby(ls.eta, step.delta.tensor, 1.0, theta.tensor),
                                theta.layout)
        book.accepted(iteration, theta, step, ls)
    trace.final_theta = theta
    return trace


def _pipelined_loop(book: _Book, rmap_provider, theta: ParameterVector, config: OptimizerConfig,
                    rng) -> ParameterVector:
    """The dense loop with iteration i+1 queued before iteration i's results are read
    (SURVEY 8f rank 1).  The line-search selection, the theta update and the
    rejection multiplier run on the device inside the iteration's CUDA graph
    (solver._DenseGraph pipe_*), so the host only books rows one step behind.
    Same trajectory as the eager loop: a factorisation failure or a non-finite
    loss (rare) discards the queued successor and redoes the iteration eagerly
    with the retry ladder before the pipeline resumes."""
    import collections

    from .solver import StepResult as _SR
    from .solver import _DenseGraph

    config_pc = config.line_search_points
    etas = 2.0 ** -np.arange(config_pc, dtype=np.float64)
    book.snapshot = True  # theta views point into the ping-pong buffers
    G = None
    pending = collections.deque()  # (iteration, rmap, ticket)
    iteration = 0
    stop = False
    fails = 0  # consecutive iterations whose first factorisation failed
    cur = theta  # theta after the last booked iteration

    def queue_next() -> bool:
        nonlocal iteration, G
        iteration += 1
        if _budget_reached(config, iteration, book.clock):
            return False
        rmap = rmap_provider(iteration)
        if G is None:
            G = _DenseGraph.get(rmap, config.use_ga, config_pc, config.lam_cap)
            G.pipe_start(cur.tensor, config.reject_if_worse)
        if not (_pipeline_ok(rmap, config) and G.pipe_matches(rmap)):
            raise _Unpipelinable(iteration, rmap)
        pending.append((iteration, rmap, G.pipe_enqueue(rmap)))
        return True

    def eager_redo(it, rmap, theta_in):
        """Iteration `it` on the host-driven path; returns (theta_after, stop)."""
        try:
            step, ls, loss = _eager_body(rmap, theta_in, config, rng, book.rejections,
                                         redo=True)
        except Exception as exc:
            book.abort(it, exc)
            return theta_in, True
        if ls.rejected or (config.reject_if_worse and ls.loss > loss):
            return theta_in, book.rejected(it, theta_in, step, ls, loss)
        from . import kernels as K

        new = ParameterVector(K.axpby(ls.eta, step.delta.tensor, 1.0, theta_in.tensor),
                              theta_in.layout)
        book.accepted(it, new, step, ls)
        return new, False

    peek = _DenseGraph.peek(rmap_provider(1), config.use_ga, config_pc, config.lam_cap)
    if peek is not None and peek.ladder_mode:
        # learned on an earlier run of this problem (per thread): every first damping
        # failed, so iterate on the retry ladder directly (same trajectory)
        book.rel_pending = None
        return _finish_eager(book, rmap_provider, theta, config, rng, 1, rmap_provider(1),
                             redo=True)
    try:
        more = queue_next()
        while pending and not stop:
            if more:
                more = queue_next()
            it, rmap, ticket = pending.popleft()
            arr, t_after, delta = G.pipe_fetch(ticket)
            book.resolve(keep=0)
            rr, lam_used, v2, a2, anyd = arr[1], arr[2], arr[3], arr[4], arr[5]
            sel = arr[6 + config_pc: 10 + config_pc]
            status = int(sel[2])
            loss = 0.5 * float(rr)
            view = ParameterVector(t_after, cur.layout)
            if status >= 2:  # failed factorisation / non-finite loss: redo eagerly
                succ = pending.popleft() if pending else None
                if succ is not None:
                    succ[2][1].synchronize()  # let the discarded successor drain
                theta_in = ParameterVector(t_after.clone(), cur.layout)
                cur, stop = eager_redo(it, rmap, theta_in)
                fails += 1
                if fails >= 2:
                    G.ladder_mode = True
                if succ is not None and not stop and fails >= 2:
                    # the first damping keeps failing (K + lam I not PD in FP64, e.g.
                    # config 4): every pipelined attempt would cost a second Gram, so
                    # the rest of the run takes the ladder on each iteration's own K
                    book.resolve()
                    book.rel_pending = None
                    return _finish_eager(book, rmap_provider, cur, config, rng, succ[0],
                                         succ[1], redo=True)
                if succ is not None and not stop:
                    G.pipe_rewind(ticket, cur.tensor, 10.0**book.rejections)
                    pending.appendleft((succ[0], succ[1], G.pipe_enqueue(succ[1])))
                continue
            fails = 0
            v_norm = float(np.sqrt(v2))
            ga = None
            if config.use_ga and v_norm > 1e-12:
                ga = 2.0 * float(np.sqrt(a2)) / v_norm
            step = _SR(delta=ParameterVector(delta, cur.layout), lambda_used=float(lam_used),
                       cg_iterations=0, ga_ratio=ga)
            if status == 1:
                losses = arr[6: 6 + config_pc]
                ls = _select(losses, etas, loss, config_pc)
                cur = view
                stop = book.rejected(it, view, step, ls, loss)
                continue
            if anyd == 0.0:
                ls = LineSearchResult(1.0, loss, False, 0, False)
            else:
                j = int(sel[3])
                ls = LineSearchResult(float(etas[j]), float(sel[1]), float(sel[1]) > loss,
                                      config_pc, False)
            cur = view
            book.accepted(it, view, step, ls)
    except _Unpipelinable as u:
        # a map the pipeline cannot run (shape change): drain and finish eagerly
        while pending:
            it, rmap, ticket = pending.popleft()
            G.pipe_fetch(ticket)
        book.resolve()
        cur = ParameterVector(cur.tensor.clone(), cur.layout)
        book.rel_pending = None
        return _finish_eager(book, rmap_provider, cur, config, rng, u.iteration, u.rmap)
    except Exception as exc:  # errors from the provider or the host bookkeeping
        book.abort(iteration, exc)
    while pending:  # stopped with a successor in flight: let it drain, ignore it
        _, _, ticket = pending.popleft()
        ticket[1].synchronize()
    book.resolve()
    return ParameterVector(cur.tensor.clone(), cur.layout)


class _Unpipelinable(Exception):
    def __init__(self, iteration, rmap):
        super().__init__(iteration)
        self.iteration, self.rmap = iteration, rmap


def _finish_eager(book, rmap_provider, theta, config, rng, iteration, rmap, redo=False):
    """The remaining iterations step by step (redo=True: straight to the retry
    ladder on each iteration's K, no fused single-attempt first)."""
    from . import kernels as K

    first = True
    while True:
        if not first:
            iteration += 1
            if _budget_reached(config, iteration, book.clock):
                break
        try:
            if not first:
                rmap = rmap_provider(iteration)
            first = False
            step, ls, loss = _eager_body(rmap, theta, config, rng, book.rejections, redo=redo)
        except Exception as exc:
            book.abort(iteration, exc)
            break
        if ls.rejected or (config.reject_if_worse and ls.loss > loss):
            if book.rejected(iteration, theta, step, ls, loss):
                break
            continue
        theta = ParameterVector(K.axpby(ls.eta, step.delta.tensor, 1.0, theta.tensor),
                                theta.layout)
        book.accepted(iteration, theta, step, ls)
    return theta


def dngd_minimize(residual_map: ResidualMap, theta, config: OptimizerConfig,
                  rng=None) -> TrainTrace:
    """optimizer.py:268-273."""
    if rng is None or isinstance(rng, (int, np.integer)):
        rng = np.random.default_rng(rng)
    if not isinstance(theta, ParameterVector):
        theta = ParameterVector(theta, residual_map.layout)
    trace = TrainTrace(problem="custom", method="dngd", seed=-1)
    from ._state import thread_stream

    with thread_stream():
        return _dngd_loop(trace, lambda it: residual_map, theta, config, rng)


# -- primal oracles and the primal/dual regime sweep -----------------


def _normal_matrix_t(rmap, theta):
    """J^T J (n x n) on the FP64 tensor cores: the SYRK of the transposed Jacobian."""
    from . import kernels as K

    J = rmap.jacobian_t(theta)
    n = rmap.n
    Jt = K.transpose_pad(J[:, :n])  # (n, m) row-major, 16-aligned pitch
    return J, K.syrk(Jt, rmap.m)


def primal_gn_solve(residual_map: ResidualMap, theta, g, points=None,
                    lam: float = 1e-3) -> ParameterVector:
    """Parameter-space damped Gauss-Newton step (J^T J + lam I) dtheta = -g
    (optimizer.py:331-346): the small-n oracle and the n << m path, with the same
    lam *= 10 retry ladder as the dual solve."""
    from .solver import _chol_with_retries

    if lam <= 0.0:
        raise DomainError(f"damping must be positive, got {lam}")
    rmap = residual_map if points is None else residual_map.rebind(points)
    if not isinstance(theta, ParameterVector):
        theta = ParameterVector(theta, rmap.layout)
    g_t = rmap._vec_t(g.tensor if isinstance(g, ParameterVector) else g, rmap.n, "gradient")
    _, JtJ = _normal_matrix_t(rmap, theta)
    fac, _ = _chol_with_retries(JtJ, lam)
    delta = fac.solve_((-g_t).contiguous())
    return ParameterVector(delta, theta.layout)


def primal_ga_correction(residual_map: ResidualMap, theta, v, points=None,
                         lam: float = 1e-3) -> ParameterVector:
    """Parameter-space geodesic acceleration (J^T J + lam I) a = -J^T f_vv
    (optimizer.py:349-362)."""
    from . import kernels as K
    from .solver import _chol_with_retries

    if lam <= 0.0:
        raise DomainError(f"damping must be positive, got {lam}")
    rmap = residual_map if points is None else residual_map.rebind(points)
    if not isinstance(theta, ParameterVector):
        theta = ParameterVector(theta, rmap.layout)
    v_t = rmap._vec_t(v.tensor if isinstance(v, ParameterVector) else v, rmap.n, "direction")
    f_vv = rmap.fvv_t(theta, v_t)
    J, JtJ = _normal_matrix_t(rmap, theta)
    fac, _ = _chol_with_retries(JtJ, lam)
    rhs = K.gemv_t(J, f_vv, rmap.n, None, -1.0)
    return ParameterVector(fac.solve_(rhs), theta.layout)


def timing_sweep(grid, iterations: int = 3, lam: float = 1e-3, seed: int = 0) -> list:
    """Mean per-step seconds of primal vs dual dense solves on random linear maps
    (optimizer.py:482-519): Gram/normal-matrix assembly, Cholesky and recovery,
    device-synchronised.  Only the relative ordering is meaningful."""
    import torch

    from .residuals import LinearResidualMap

    rng = np.random.default_rng(seed)
    rows = []
    for m, n in grid:
        A = rng.normal(size=(m, n)) / np.sqrt(n)
        rmap = LinearResidualMap(A, rng.normal(size=m))
        theta = ParameterVector(rng.normal(size=n), rmap.layout)
        primal_times, dual_times = [], []
        for _ in range(iterations):
            torch.cuda.current_stream().synchronize()
            t0 = time.perf_counter()
            g = rmap.gradient_t(theta)
            primal_gn_solve(rmap, theta, g, lam=lam)
            torch.cuda.current_stream().synchronize()
            primal_times.append(time.perf_counter() - t0)
            t0 = time.perf_counter()
            g = rmap.gradient_t(theta)
            dense_dual_solve(rmap, theta, g, lam=lam, use_ga=False)
            torch.cuda.current_stream().synchronize()
            dual_times.append(time.perf_counter() - t0)
        primal_s = float(np.mean(primal_times))
        dual_s = float(np.mean(dual_times))
        rows.append({"m": m, "n": n, "primal_s": primal_s, "dual_s": dual_s,
                     "winner": "dual" if dual_s < primal_s else "primal"})
    return rows


def relative_l2_error(u_pred, u_exact) -> float:
    """optimizer.py:465-477."""
    u_pred = np.asarray(u_pred, dtype=np.float64).reshape(-1)
    u_exact = np.asarray(u_exact, dtype=np.float64).reshape(-1)
    if u_pred.shape != u_exact.shape:
        raise DomainError(f"prediction and reference shapes differ: {u_pred.shape} vs {u_exact.shape}")
    denom = float(np.linalg.norm(u_exact))
    if denom == 0.0:
        raise DomainError("reference values are identically zero on the grid")
    return float(np.linalg.norm(u_pred - u_exact)) / denom


class _ValueProblem:
    """u(x) - u*(x) as a one-class residual map: the rel-L2 metric on the device.
    Carries the problem's input embedding and output transform (model.py:133-277):
    u = factor(x) * phi(embedding(x))."""

    def __init__(self, dim, exact, problem=None):
        self.raw_dim = dim
        self.exact = exact
        self.problem = problem
        self.input_dim = getattr(problem, "input_dim", dim) if problem is not None else dim
        if problem is not None and hasattr(problem, "value_factor"):
            self.point_coefs = self._coefs
        tr = getattr(problem, "transform", None)
        if tr is not None and tr.kind == "ic_shift":
            self.transform = tr  # u = phi - phi(0, .) + q0 on the grid too (model.py:237-248)

    def class_operator(self, class_id):
        from .problems import VALUE

        return VALUE

    def class_data(self, cls):
        return self.exact

    def input_channels(self, cls, op):
        if self.problem is None or not hasattr(self.problem, "input_channels"):
            return None
        return self.problem.input_channels(cls, op)

    def _coefs(self, cls, op):
        return self.problem.value_factor(cls.points)[:, None]


def _rel_l2_fn(problem, spec: MlpSpec):
    """Relative L2 error on the problem's evaluation grid (optimizer.py:282-287)."""
    if not getattr(problem, "has_exact", False):
        return None
    from .residuals import INTERIOR, CollocationClass, CollocationSet

    pts = problem.eval_points()
    exact = problem.exact_solution(pts)
    denom = float(np.linalg.norm(exact))
    vmap = PinnResidualMap(_ValueProblem(pts.shape[1], exact, problem), spec,
                           CollocationSet([CollocationClass(INTERIOR, pts, 1.0)]))

    def fn(theta):
        if denom == 0.0:
            raise DomainError("reference values are identically zero on the grid")
        r = vmap.residuals_t(theta)
        return float(r.norm().item()) / denom

    def enqueue(theta):
        """Queue the evaluation (no host sync); fetch() reads it later."""
        import torch

        if denom == 0.0:
            raise DomainError("reference values are identically zero on the grid")
        nrm = vmap.residuals_t(theta).norm().reshape(1)
        host = torch.empty(1, dtype=torch.float64, pin_memory=True)
        host.copy_(nrm, non_blocking=True)
        ev = torch.cuda.Event()
        ev.record()
        return host, ev

    def fetch(handle):
        host, ev = handle
        ev.synchronize()
        return float(host[0]) / denom

    fn.enqueue, fn.fetch = enqueue, fetch
    return fn


def network_values(problem, spec: MlpSpec, theta, pts) -> np.ndarray:
    """Network output on raw points (optimizer.py:276-279)."""
    from .residuals import INTERIOR, CollocationClass, CollocationSet

    pts = np.asarray(pts, dtype=np.float64)
    vmap = PinnResidualMap(_ValueProblem(pts.shape[1], np.zeros(pts.shape[0]), problem), spec,
                           CollocationSet([CollocationClass(INTERIOR, pts, 1.0)]))
    return vmap.residuals_t(theta).cpu().numpy()


def dngd_run(problem, spec: MlpSpec, config: OptimizerConfig, seed: int, counts=None,
             init: str = "glorot_uniform", track_rel_l2: bool = True, on_step=None,
             gram_shard=None) -> TrainTrace:
    """Train a network on a PDE problem with D-NGD (optimizer.py:290-314).

    `init` selects the initialiser ("glorot_uniform" = reference default,
    "xavier_normal" = BASELINE configs); the seed drives the initialisation and
    every collocation / landmark draw in the reference's order.  gram_shard =
    (comm, rank, world) splits the factored Gram's tiles over the ranks (one K
    all-reduce per step; everything else replicated -- SURVEY §8e).
    """
    from .problems import sample_collocation

    spec = replace(spec, seed=seed)
    rng = np.random.default_rng(seed)
    theta = INITIALIZERS[init](spec)
    state = {"rmap": None}

    def provider(iteration: int) -> ResidualMap:
        if state["rmap"] is None or (config.resample and iteration > 1):
            colloc = sample_collocation(problem, counts, rng)
            if state["rmap"] is None:
                state["rmap"] = PinnResidualMap(problem, spec, colloc)
                state["rmap"].gram_shard = gram_shard
            else:
                state["rmap"] = state["rmap"].rebind(colloc)
        return state["rmap"]

    trace = TrainTrace(problem=problem.name, method="dngd", seed=seed)
    from ._state import thread_stream

    with thread_stream():  # off the main thread: this thread's own stream
        rel_fn = _rel_l2_fn(problem, spec) if track_rel_l2 else None
        return _dngd_loop(trace, provider, theta, config, rng, rel_fn, on_step)
