"""Residual maps with device-resident Jacobians (reference residuals.py:1-454).

The plugin contract is the reference's `ResidualMap`: `n`, `m`, `partition`,
`residual_batch`, `loss`, `loss_many`, `vjp`, `residuals_and_gradient`,
`linearize`, `jacobian`, `rows_jacobian`, `jvp`, `jvp_many`,
`second_directional`, `sub_map`, `rebind`.  Those names keep returning
host numpy arrays for drop-in callers.  The solver uses the device API
(`*_t` methods) that every map here implements on CUDA tensors:

  linearize_t(theta) -> (r, J)   J is (m, ldJ) row-major, columns [:n] valid
  fvv_t(theta, v)                f_vv = d^2/dt^2 r(theta + t v)
  losses_along_t(theta, d, etas) 0.5 |r(theta + eta_c d)|^2 for every eta_c

PinnResidualMap runs entirely in the CUDA library (pinn.cu): one
forward-Laplacian pass + per-point adjoint writes r and J, the Jacobian is
cached per parameter version so residuals_and_gradient followed by the step
assembles J once (the reference assembles it twice).
"""

from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np

from .errors import DimensionError, DomainError, NonFiniteError
from .params import ParameterLayout, ParameterVector
from .timing import stage

INTERIOR = "interior"
BOUNDARY = "boundary"
INITIAL = "initial"
_CLASS_IDS = (INTERIOR, BOUNDARY, INITIAL)


@dataclass
class CollocationClass:
    """Points of one residual class with its loss weight (residuals.py:33-55)."""

    class_id: str
    points: np.ndarray
    weight: float
    aux: dict = field(default_factory=dict)

    def __post_init__(self):
        if self.class_id not in _CLASS_IDS:
            raise DimensionError(f"unknown residual class id: {self.class_id!r}")
        pts = np.asarray(self.points, dtype=np.float64)
        self.points = pts[:, None] if pts.ndim == 1 else pts

    @property
    def count(self) -> int:
        return self.points.shape[0]


class CollocationSet:
    """Ordered residual classes; rows of r follow this order (residuals.py:58-104)."""

    def __init__(self, classes: list[CollocationClass]):
        if not classes:
            raise DimensionError("a collocation set needs at least one class")
        self.classes = list(classes)

    @property
    def m(self) -> int:
        return sum(c.count for c in self.classes)

    def partition(self) -> list[tuple[str, int, int]]:
        spans, start = [], 0
        for c in self.classes:
            spans.append((c.class_id, start, start + c.count))
            start += c.count
        return spans

    def locate(self, row: int) -> tuple[int, int]:
        if not 0 <= row < self.m:
            raise DimensionError(f"residual row {row} out of range [0, {self.m})")
        for k, (_, start, stop) in enumerate(self.partition()):
            if row < stop:
                return k, row - start
        raise AssertionError("unreachable")

    def subset(self, rows: np.ndarray) -> "CollocationSet":
        rows = np.asarray(rows, dtype=np.int64)
        if rows.ndim != 1 or rows.size == 0:
            raise DimensionError("subset needs a non-empty 1-d list of rows")
        if np.any(np.diff(rows) <= 0):
            raise DimensionError("subset rows must be strictly increasing")
        if rows[0] < 0 or rows[-1] >= self.m:
            raise DimensionError(f"subset rows out of range [0, {self.m})")
        classes = []
        for c, (_, start, stop) in zip(self.classes, self.partition()):
            local = rows[(rows >= start) & (rows < stop)] - start
            if local.size == 0:
                continue
            aux = {k: np.asarray(v)[local] for k, v in c.aux.items()}
            classes.append(CollocationClass(c.class_id, c.points[local], c.weight, aux))
        return CollocationSet(classes)


def _is_tensor(x) -> bool:
    return type(x).__module__.startswith("torch")


class ResidualBatch:
    """Stacked residual values with their class partition (residuals.py:107-122)."""

    def __init__(self, values, partition):
        self._t = values if _is_tensor(values) else None
        self._np = None if _is_tensor(values) else np.asarray(values, dtype=np.float64)
        self.partition = partition

    @property
    def values(self) -> np.ndarray:
        if self._np is None:
            self._np = self._t.cpu().numpy()
        return self._np

    @property
    def tensor(self):
        if self._t is None:
            import torch

            from ._lib import require_cuda

            self._t = torch.as_tensor(self._np, device=require_cuda())
        return self._t

    @property
    def m(self) -> int:
        return self.values.shape[0] if self._t is None else self._t.shape[0]

    def per_class(self) -> dict[str, np.ndarray]:
        return {cid: self.values[a:b] for cid, a, b in self.partition}

    def loss(self) -> float:
        if self._t is not None:
            from . import kernels as K

            return 0.5 * float(K.dot(self._t, self._t).item())
        return 0.5 * float(self.values @ self.values)


def _raise_nonfinite(values_t, partition):
    """NonFiniteError naming the class and point of the first non-finite residual
    (residuals.py:125-136), found by the device scan dngd_nonfinite_report."""
    from . import kernels as K

    hit = K.nonfinite_report(values_t.contiguous(), [b for _, _, b in partition])
    if hit is None:
        return
    k, point = hit
    if 0 <= k < len(partition):
        cid = partition[k][0]
        raise NonFiniteError(
            f"non-finite residual in class {cid!r} at point {point}",
            class_id=cid,
            point_index=point,
        )
    raise NonFiniteError("non-finite residual", point_index=point)


class ResidualMap:
    """Device-first residual map base class."""

    layout: ParameterLayout
    collocation: CollocationSet

    # -- shapes --------------------------------------------------------------------
    @property
    def n(self) -> int:
        return self.layout.size

    @property
    def m(self) -> int:
        return self.collocation.m

    def partition(self):
        return self.collocation.partition()

    def rebind(self, collocation: CollocationSet) -> "ResidualMap":
        raise NotImplementedError

    def sub_map(self, rows: np.ndarray) -> "ResidualMap":
        return self.rebind(self.collocation.subset(rows))

    def _theta_t(self, theta):
        if isinstance(theta, ParameterVector):
            if theta.layout != self.layout:
                raise DimensionError("parameter vector layout does not match this map")
            return theta.tensor
        if _is_tensor(theta):
            return theta
        return ParameterVector(np.asarray(theta, dtype=np.float64), self.layout).tensor

    def _vec_t(self, v, size, what):
        import torch

        from ._lib import require_cuda

        if isinstance(v, ParameterVector):
            v = v.tensor
        elif isinstance(v, ResidualBatch):
            v = v.tensor
        if not _is_tensor(v):
            v = torch.as_tensor(np.ascontiguousarray(v, dtype=np.float64), device=require_cuda())
        if v.dim() != 1 or v.shape[0] != size:
            raise DimensionError(f"{what} has shape {tuple(v.shape)}, expected ({size},)")
        return v.contiguous()

    # -- device API (subclasses implement linearize_t / fvv_t / losses) -------------
    def linearize_t(self, theta):
        raise NotImplementedError

    def residuals_t(self, theta):
        return self.linearize_t(theta)[0]

    def jacobian_t(self, theta):
        return self.linearize_t(theta)[1]

    def fvv_t(self, theta, v_t):
        raise NotImplementedError

    def loss_many_t(self, cands_t):
        raise NotImplementedError

    def losses_along_t(self, theta, delta_t, etas_t):
        th = self._theta_t(theta)
        cands = th[None, :] + etas_t[:, None] * delta_t[None, :]
        return self.loss_many_t(cands)

    def jvp_t(self, theta, v_t):
        from . import kernels as K

        return K.gemv_n(self.jacobian_t(theta), v_t, self.n)

    def vjp_t(self, theta, w_t, g_t=None, scale=1.0):
        from . import kernels as K

        return K.gemv_t(self.jacobian_t(theta), w_t, self.n, g_t, scale)

    def gradient_t(self, theta):
        r, J = self.linearize_t(theta)
        from . import kernels as K

        return K.gemv_t(J, r, self.n)

    # -- reference (numpy) API --------------------------------------------------------
    def residual_batch(self, theta) -> ResidualBatch:
        r = self.residuals_t(theta)
        _raise_nonfinite(r, self.partition())
        return ResidualBatch(r, self.partition())

    def loss(self, theta) -> float:
        return self.residual_batch(theta).loss()

    def loss_many(self, candidates) -> np.ndarray:
        import torch

        from ._lib import require_cuda

        if not _is_tensor(candidates):
            candidates = np.asarray(candidates, dtype=np.float64)
            if candidates.ndim != 2:
                raise DimensionError("loss_many expects a (C, n) candidate stack")
            candidates = torch.as_tensor(candidates, device=require_cuda())
        return self.loss_many_t(candidates.contiguous()).cpu().numpy()

    def vjp(self, theta, w) -> np.ndarray:
        return self.vjp_t(theta, self._vec_t(w, self.m, "cotangent")).cpu().numpy()

    def residuals_and_gradient(self, theta):
        r, J = self.linearize_t(theta)
        loss = 0.5 * float((r @ r).item())
        if not np.isfinite(loss):
            _raise_nonfinite(r, self.partition())
        from . import kernels as K

        g = K.gemv_t(J, r, self.n)
        return ResidualBatch(r, self.partition()), g.cpu().numpy()

    def gradient(self, theta) -> np.ndarray:
        return self.residuals_and_gradient(theta)[1]

    def linearize(self, theta):
        r, J = self.linearize_t(theta)
        _raise_nonfinite(r, self.partition())
        return ResidualBatch(r, self.partition()), J[:, : self.n].cpu().numpy()

    def jacobian(self, theta) -> np.ndarray:
        return self.linearize(theta)[1]

    def rows_jacobian(self, theta, rows) -> np.ndarray:
        return self.sub_map(rows).jacobian(theta)

    def jvp(self, theta, v) -> np.ndarray:
        return self.jvp_t(theta, self._vec_t(v, self.n, "tangent")).cpu().numpy()

    def jvp_many(self, theta, tangents) -> np.ndarray:
        import torch

        from . import kernels as K
        from ._lib import require_cuda

        V = np.asarray(tangents, dtype=np.float64)
        if V.ndim != 2 or V.shape[1] != self.n:
            raise DimensionError(f"tangent has shape {V.shape}, expected (..., {self.n})")
        J = self.jacobian_t(theta)
        Vd = torch.zeros((V.shape[0], J.shape[1]), dtype=torch.float64, device=require_cuda())
        Vd[:, : self.n] = torch.as_tensor(V, device=Vd.device)
        return K.gemm_nt(Vd, J, K=self.n).cpu().numpy()

    def second_directional(self, theta, v) -> np.ndarray:
        f = self.fvv_t(theta, self._vec_t(v, self.n, "tangent"))
        _raise_nonfinite(f, self.partition())
        return f.cpu().numpy()


class LinearResidualMap(ResidualMap):
    """r(theta) = A theta + c (residuals.py:325-379); J = A on the device."""

    def __init__(self, A, c):
        self.A = np.atleast_2d(np.asarray(A, dtype=np.float64))
        self.c = np.asarray(c, dtype=np.float64)
        if self.c.shape != (self.A.shape[0],):
            raise DimensionError(f"offset has shape {self.c.shape}, expected ({self.A.shape[0]},)")
        self.layout = ParameterLayout([("theta", (self.A.shape[1],))])
        self.collocation = CollocationSet(
            [CollocationClass(INTERIOR, np.arange(self.A.shape[0])[:, None] * 1.0, 1.0)]
        )
        self._dev = None

    def rebind(self, collocation):
        rows = collocation.classes[0].points[:, 0].astype(np.int64)
        sub = LinearResidualMap(self.A[rows], self.c[rows])
        sub.layout = self.layout
        return sub

    def _device(self):
        if self._dev is None:
            import torch

            from . import kernels as K
            from ._lib import require_cuda

            m, n = self.A.shape
            J = torch.zeros((m, K.pad_ld(n)), dtype=torch.float64, device=require_cuda())
            J[:, :n] = torch.as_tensor(self.A, device=J.device)
            self._dev = (J, torch.as_tensor(self.c, device=J.device))
        return self._dev

    def linearize_t(self, theta):
        from . import kernels as K

        J, c = self._device()
        r = K.gemv_n(J, self._theta_t(theta), self.n, 1.0, c, 1.0)
        return r, J

    def fvv_t(self, theta, v_t):
        import torch

        return torch.zeros(self.m, dtype=torch.float64, device=v_t.device)

    def loss_many_t(self, cands_t):
        import torch

        from . import kernels as K

        J, c = self._device()
        C = cands_t.shape[0]
        Cd = torch.zeros((C, J.shape[1]), dtype=torch.float64, device=J.device)
        Cd[:, : self.n] = cands_t
        R = K.gemm_nt(Cd, J, K=self.n) + c[None, :]
        return 0.5 * (R * R).sum(dim=1)


def _act_state() -> dict:
    """Which (theta version, map) this thread's activation workspace holds."""
    from ._state import tls

    return tls().act_state


def _upload(arr, dev):
    """Host array -> device through pinned staging, queued on the current stream
    without a host-side stream sync (a pageable copy would wait for the queued
    work, which stalls the pipelined loop while it samples the next collocation)."""
    import torch

    t = torch.from_numpy(np.ascontiguousarray(arr))
    return t.pin_memory().to(dev, non_blocking=True)


class PinnResidualMap(ResidualMap):
    """Weighted PDE residuals of a tanh MLP, evaluated by the CUDA library."""

    LOSS_WS_BUDGET = 8 * 1024**3  # bytes of line-search activations per chunk

    def __new__(cls, *args, **kwargs):
        # problems with the ic_shift output transform get the two-map form
        if cls is PinnResidualMap:
            problem = args[0] if args else kwargs.get("problem")
            if _is_ic_shift(problem):
                return IcShiftResidualMap(*args, **kwargs)
        return super().__new__(cls)

    def __init__(self, problem, spec, collocation: CollocationSet, col_range=None):
        from .model import MlpSpec

        if not isinstance(spec, MlpSpec):
            raise DimensionError("PinnResidualMap needs an MlpSpec")
        in_dim = getattr(problem, "input_dim", problem.raw_dim)
        if spec.input_dim != in_dim:
            raise DimensionError(
                f"spec input width {spec.input_dim} != problem input width {in_dim}"
            )
        if spec.output_dim != 1:
            raise DimensionError("PINN residual maps need a scalar network output")
        self.problem = problem
        self.spec = spec
        self.layout = spec.layout()
        self.collocation = collocation
        self.col_range = (0, self.layout.size) if col_range is None else tuple(col_range)
        self._dev = None
        self._cache = None
        self._rcache = None
        self._J = None

    def rebind(self, collocation):
        other = PinnResidualMap(self.problem, self.spec, collocation, self.col_range)
        other.gram_shard = self.gram_shard
        if self._J is not None and self._J.shape[0] == collocation.m:
            other._J = self._J  # reuse the Jacobian buffer across resamples
            self._cache = None  # this map no longer owns the buffer contents
        return other

    # -- device state -----------------------------------------------------------------
    def _device(self):
        if self._dev is not None:
            return self._dev
        import torch

        from . import _lib
        from . import kernels as K
        from ._lib import require_cuda

        dev = require_cuda()
        classes = self.collocation.classes
        if len(classes) > _lib.MAX_CLASSES:
            raise DomainError(f"at most {_lib.MAX_CLASSES} residual classes are supported")
        if self.m > 65535:
            raise DomainError("at most 65535 residual rows per map in this build")
        arr = (_lib.ClassDesc * len(classes))()
        keep = []
        for k, cls in enumerate(classes):
            op = self.problem.class_operator(cls.class_id)
            pts = _upload(cls.points, dev)
            f = _upload(np.asarray(self.problem.class_data(cls), dtype=np.float64), dev)
            keep += [pts, f]
            d = arr[k]
            d.count = cls.count
            d.ngrad = len(op.grad_dims)
            d.nlap = len(op.lap_dims)
            if d.ngrad > _lib.MAX_GRAD:
                raise DomainError("too many derivative channels for the device kernels")
            for g, gd in enumerate(op.grad_dims):
                d.grad_dims[g] = int(gd)
                d.cg[g] = float(op.cg[g])
            for l, ldim in enumerate(op.lap_dims):
                d.lap_grad[l] = op.grad_dims.index(ldim)
            d.cu, d.cl, d.weight = float(op.cu), float(op.cl), float(cls.weight)
            d.c3 = float(getattr(op, "c3", 0.0))
            d.points = pts.data_ptr()
            d.f = f.data_ptr()
            emb = (self.problem.input_channels(cls, op)
                   if hasattr(self.problem, "input_channels") else None)
            if emb is not None:
                emb = np.ascontiguousarray(emb, dtype=np.float64)
                if emb.shape != (cls.count, 1 + d.ngrad + (1 if d.nlap else 0),
                                 self.spec.input_dim):
                    raise DimensionError(f"input channels of class {cls.class_id}: {emb.shape}")
                inp = _upload(emb, dev)
                keep.append(inp)
                d.inputs = inp.data_ptr()
            if hasattr(self.problem, "point_grad_dims"):  # per-point derivative dims (STDE)
                gi = np.ascontiguousarray(self.problem.point_grad_dims(cls), dtype=np.int32)
                if gi.shape != (cls.count, d.ngrad):
                    raise DimensionError(f"point derivative dims of class {cls.class_id}: {gi.shape}")
                gi_t = _upload(gi, dev)
                keep.append(gi_t)
                d.grad_idx = gi_t.data_ptr()
            if hasattr(self.problem, "point_coefs"):  # per-point coefficients
                co = np.ascontiguousarray(self.problem.point_coefs(cls, op), dtype=np.float64)
                if co.shape != (cls.count, 1 + d.ngrad + (1 if d.nlap else 0)):
                    raise DimensionError(f"point coefficients of class {cls.class_id}: {co.shape}")
                co_t = _upload(co, dev)
                keep.append(co_t)
                d.coefs = co_t.data_ptr()
        mlp = K.mlp_desc(self.spec.layer_widths)
        ws_bytes = K.pinn_workspace_bytes(mlp, arr, len(classes), 1)
        # line-search activations grow linearly with the candidate count
        per_cand = (K.pinn_workspace_bytes(mlp, arr, len(classes), 64)
                    - K.pinn_workspace_bytes(mlp, arr, len(classes), 32)) // 32
        self._dev = dict(arr=arr, keep=keep, mlp=mlp, nclass=len(classes), ws_bytes=ws_bytes,
                         per_cand=max(per_cand, 1), device=dev)
        return self._dev

    def _workspace(self, nbytes, tag="pinn_scratch"):
        """Scratch for f_vv / line search / residual-only passes."""
        from . import kernels as K

        return K.workspace(tag, nbytes)

    def _act_workspace(self):
        """Activation workspace (forward channels + adjoints of the last assembly):
        kept apart from the scratch so J^T w can reuse it after f_vv / line search."""
        from . import kernels as K

        return K.workspace("pinn_act", self._device()["ws_bytes"])

    @property
    def ncols(self) -> int:
        return self.col_range[1] - self.col_range[0]

    def _key(self, th):
        return (th.data_ptr(), th._version, id(self.collocation))

    def linearize_t(self, theta):
        import torch

        from . import kernels as K

        th = self._theta_t(theta)
        key = self._key(th)
        if self._cache is not None and self._cache[0] == key:
            return self._cache[1], self._cache[2]
        d = self._device()
        m = self.m
        if self._J is None or self._J.shape != (m, K.pad_ld(self.ncols)):
            self._J = torch.empty((m, K.pad_ld(self.ncols)), dtype=torch.float64, device=d["device"])
        r = torch.empty(m, dtype=torch.float64, device=d["device"])
        with stage("assemble"):
            K.assemble(d["mlp"], th, d["arr"], d["nclass"], r, self._J, self.col_range[0],
                       self.col_range[1], self._act_workspace())
        _act_state()["key"] = (key, self._act_identity())
        _act_state()["theta"] = th  # keeps the keyed storage alive (no address reuse)
        self._cache = (key, r, self._J, th)
        return r, self._J

    def residuals_t(self, theta):
        import torch

        from . import kernels as K

        th = self._theta_t(theta)
        if self._cache is not None and self._cache[0] == self._key(th):
            return self._cache[1]
        if self._rcache is not None and self._rcache[0] == self._key(th):
            return self._rcache[1]
        d = self._device()
        r = torch.empty(self.m, dtype=torch.float64, device=d["device"])
        K.assemble(d["mlp"], th, d["arr"], d["nclass"], r, None, 0, self.n,
                   self._workspace(d["ws_bytes"]))
        return r

    def fvv_t(self, theta, v_t):
        import torch

        from . import kernels as K

        d = self._device()
        out = torch.empty(self.m, dtype=torch.float64, device=d["device"])
        th = self._theta_t(theta)
        with stage("fvv"):
            K.fvv(d["mlp"], th, v_t, d["arr"], d["nclass"], out, self._workspace(d["ws_bytes"]),
                  self._reuse_act(th))
        return out

    def _reuse_act(self, th):
        """The activation workspace when it holds the pass at theta and the input
        layer is wide (x W0 is then reused by f_vv and the line search)."""
        if self.spec.input_dim >= 64 and self.wide_input() and self._act_valid(th):
            return self._act_workspace()
        return None

    # -- factored Gram and J^T w (no pass over J) ----------------------------------------
    gram_mode = "auto"  # "auto" | "factored" | "materialized"

    def _gram_flop_ratio(self) -> float:
        """Estimated FLOPs of the factored Gram (executed: whole 64-row tiles of
        floor(64/nch) packed points, 16-column K chunks) / FLOPs of J J^T."""
        ksum = self._gram_ksum(chunked=True)
        fact = 0.0
        for c in self.collocation.classes:
            for cp in self.collocation.classes:
                fact += self._tile_rows(c) * self._tile_rows(cp) * ksum
        return fact / max(1.0, float(self.m) ** 2 * self.n)

    def _tile_rows(self, cls) -> int:
        """G-space rows the packed kernel runs for a class: 64 per floor(64/nch) points."""
        ppt = max(1, 64 // self._nch(cls))
        return -(-cls.count // ppt) * 64

    def factored_gram_flops(self, executed: bool = False) -> float:
        """FLOPs of the factored Gram.  Useful (default): the lower triangle of the
        point pairs x nch_c nch_c' channel pairs x the two GEMM K-dims per layer
        (w_k for G^H, w_{k+1} for G^Z; the output layer's Zbar are seeds) -- the
        work of the algorithm with nothing padded.  executed=True: what the kernel
        issues (whole 64-row tiles, 16-column K chunks)."""
        ksum = self._gram_ksum(chunked=executed)
        classes = self.collocation.classes
        pairs = 0.0
        for i, c in enumerate(classes):
            for cp in classes[: i + 1]:
                if executed:
                    a, b = self._tile_rows(c) // 64, self._tile_rows(cp) // 64
                    pairs += (a * (a + 1) / 2 if cp is c else a * b) * 64 * 64
                else:
                    a, b = self._nch(c), self._nch(cp)
                    pairs += (c.count * (c.count + 1) / 2 * a * a if cp is c
                              else c.count * cp.count * a * b)
        return 2.0 * pairs * ksum

    def _gram_ksum(self, chunked: bool = True) -> int:
        """Sum over layers of the two GEMM K-dims (in the kernel's 16-column chunks
        when chunked)."""
        w = self.spec.layer_widths
        c16 = (lambda x: -(-x // 16) * 16) if chunked else (lambda x: x)  # noqa: E731
        return sum(c16(w[k]) + (c16(w[k + 1]) if k <= len(w) - 3 else 0)
                   for k in range(len(w) - 1))

    def _nch(self, cls) -> int:
        op = self.problem.class_operator(cls.class_id)
        return 1 + len(op.grad_dims) + (1 if op.lap_dims else 0)

    def wide_input(self) -> bool:
        """Raw (identity) inputs wider than the channel kernels (din > 12, the STDE
        case): the J-free Gram forms J's input block from X X^T and the input-layer
        adjoints, and only the hidden/output columns are materialised (pinn.cu
        gram_wide_input)."""
        from . import _lib

        return self.spec.input_dim > _lib.MAX_GRAD and all(
            not d.inputs for d in self._device()["arr"])

    def use_factored_gram(self) -> bool:
        if self.col_range != (0, self.layout.size):
            return False  # column shards form their partial Gram from J_p
        if self.wide_input():
            # the input block is (din+1) w1 of n columns: never worth writing J
            return self.gram_mode != "materialized" and self.gram_shard is None
        if any(self._nch(c) > 8 for c in self.collocation.classes):
            return False
        if self.gram_mode == "factored":
            return True
        if self.gram_mode == "materialized":
            return False
        # measured crossover: heat1d (ratio ~0.5) 1.7x faster factored, poisson2d
        # (ratio > 1) slower; the J-free step also skips J's write and read
        return self._gram_flop_ratio() < 0.6

    def jfree(self) -> bool:
        """Dense step without J: factored Gram + J^T w from the activations."""
        return self.use_factored_gram()

    def jfree_pcg(self) -> bool:
        """PCG without J: J^T w / J v from activations and forward tangents, the
        Nystrom columns K[:, I] from the factored kernel (linear operators only)."""
        return self.use_factored_gram() and not self.wide_input() and all(
            float(getattr(self.problem.class_operator(c.class_id), "c3", 0.0)) == 0.0
            for c in self.collocation.classes)

    def residuals_act_t(self, theta):
        """r together with the activations (left for vjp_t / kcols_t; no J)."""
        import torch

        from . import kernels as K

        d = self._device()
        th = self._theta_t(theta)
        key = self._key(th)
        if self._act_valid(th):  # left by this theta's activation pass or assembly
            for cache in (self._rcache, self._cache):
                if cache is not None and cache[0] == key:
                    return cache[1]
        r = torch.empty(self.m, dtype=torch.float64, device=d["device"])
        with stage("activations"):
            K.activations(d["mlp"], th, d["arr"], d["nclass"], r, self._act_workspace())
        _act_state()["key"] = (key, self._act_identity())
        _act_state()["theta"] = th
        self._rcache = (key, r, th)
        return r

    def jvp_t(self, theta, v_t):
        """J v: over the cached J, else from first-order forward tangents (no J)."""
        from . import kernels as K

        th = self._theta_t(theta)
        if (self._cache is not None and self._cache[0] == self._key(th)) or not self.jfree():
            return super().jvp_t(theta, v_t)
        import torch

        d = self._device()
        out = torch.empty(self.m, dtype=torch.float64, device=d["device"])
        with stage("jvp"):
            K.jvp_factored(d["mlp"], th, v_t.contiguous(), d["arr"], d["nclass"], out,
                           self._workspace(d["ws_bytes"]))
        return out

    def kcols_t(self, theta, landmarks):
        """K[:, landmarks] (m x ell) from the activations of theta (no J)."""
        import torch

        from . import kernels as K

        d = self._device()
        self.residuals_act_t(theta)  # activations of this theta
        Kc = torch.empty((self.m, max(len(landmarks), 1) + (len(landmarks) % 2)),
                         dtype=torch.float64, device=d["device"])
        with stage("kcols"):
            K.gram_factored_cols(d["mlp"], d["arr"], d["nclass"], landmarks, Kc,
                                 self._act_workspace())
        return Kc[:, : len(landmarks)]

    def _act_identity(self):
        return (id(self), self._dev["arr"] if self._dev else None)

    def _act_valid(self, th) -> bool:
        return _act_state().get("key") == (self._key(th), self._act_identity())

    gram_shard = None  # (comm, rank, world): tile-sharded Gram summed over the ranks

    def gram_factored_t(self, theta, K_out):
        """K = J J^T (and r) from the activations; leaves them for vjp_t.  With
        gram_shard set, this rank computes 1/world of the K tiles and the parts are
        summed with one all-reduce (one reduction per Gram)."""
        import torch

        from . import kernels as K

        d = self._device()
        th = self._theta_t(theta)
        if self.wide_input():  # analytic input block: one call does activations + K
            r = torch.empty(self.m, dtype=torch.float64, device=d["device"])
            K.gram_factored(d["mlp"], th, d["arr"], d["nclass"], r, K_out, self._act_workspace())
            _act_state()["key"] = (self._key(th), self._act_identity())
            _act_state()["theta"] = th
            self._rcache = (self._key(th), r, th)
            return K_out
        self.residuals_act_t(theta)  # r + activations (stage "activations")
        ws = self._act_workspace()
        if self.gram_shard is not None:
            comm, rank, world = self.gram_shard
            K_out.zero_()
            with stage("gram_kernel"):
                K.gram_factored_act(d["mlp"], d["arr"], d["nclass"], K_out, ws, rank, world)
            if K_out.is_contiguous():
                comm.allreduce_sum_(K_out)
            else:
                tmp = comm.allreduce_sum_(K_out.contiguous())
                K_out.copy_(tmp)
        else:
            with stage("gram_kernel"):
                K.gram_factored_act(d["mlp"], d["arr"], d["nclass"], K_out, ws)
        return K_out

    def residuals_gram_t(self, theta, K_out):
        self.gram_factored_t(theta, K_out)
        return self._rcache[1], K_out

    def vjp_t(self, theta, w_t, g_t=None, scale=1.0):
        """scale * (J^T w + g); from the activations when no J is materialised."""
        from . import kernels as K

        th = self._theta_t(theta)
        if self._cache is not None and self._cache[0] == self._key(th):
            return K.gemv_t(self._J, w_t, self.ncols, g_t, scale)
        if self.col_range != (0, self.layout.size):
            return super().vjp_t(theta, w_t, g_t, scale)
        import torch

        d = self._device()
        if not self._act_valid(th):
            r = torch.empty(self.m, dtype=torch.float64, device=d["device"])
            K.activations(d["mlp"], th, d["arr"], d["nclass"], r, self._act_workspace())
            _act_state()["key"] = (self._key(th), self._act_identity())
            _act_state()["theta"] = th
            self._rcache = (self._key(th), r, th)
        out = torch.empty(self.n, dtype=torch.float64, device=d["device"])
        scratch = K.workspace("jt", K.jt_workspace_bytes(d["mlp"], d["arr"], d["nclass"]))
        with stage("vjp"):
            K.jt_factored(d["mlp"], d["arr"], d["nclass"], w_t.contiguous(), scale, out,
                          self._act_workspace(), scratch)
        if g_t is not None:
            out.add_(g_t, alpha=scale)
        return out

    def _loss_ws(self, C):
        from . import kernels as K

        d = self._device()
        return K.pinn_workspace_bytes(d["mlp"], d["arr"], d["nclass"], C)

    def _chunk(self, C):
        d = self._device()
        return max(1, min(C, int(self.LOSS_WS_BUDGET // d["per_cand"])))

    def losses_along_t(self, theta, delta_t, etas_t):
        import torch

        from . import kernels as K

        d = self._device()
        th = self._theta_t(theta)
        C = etas_t.shape[0]
        out = torch.empty(C, dtype=torch.float64, device=d["device"])
        step = self._chunk(C)
        with stage("line_search"):
            for c0 in range(0, C, step):
                c1 = min(C, c0 + step)
                ws = self._workspace(self._loss_ws(c1 - c0))
                K.loss_many(d["mlp"], th, delta_t, etas_t[c0:c1], c1 - c0, d["arr"],
                            d["nclass"], out[c0:c1], ws, self._reuse_act(th))
        return out

    def loss_many_t(self, cands_t):
        import torch

        from . import kernels as K

        d = self._device()
        if cands_t.dim() != 2 or cands_t.shape[1] != self.n:
            raise DimensionError("loss_many expects a (C, n) candidate stack")
        C = cands_t.shape[0]
        out = torch.empty(C, dtype=torch.float64, device=d["device"])
        step = self._chunk(C)
        for c0 in range(0, C, step):
            c1 = min(C, c0 + step)
            ws = self._workspace(self._loss_ws(c1 - c0))
            K.loss_many(d["mlp"], cands_t[c0:c1].contiguous(), None, None, c1 - c0, d["arr"],
                        d["nclass"], out[c0:c1], ws)
        return out


class RegressionResidualMap(PinnResidualMap):
    """r_i = weight (u_theta(x_i) - y_i) (residuals.py:382-419) as a value-only PINN class."""

    class _RegressionProblem:
        name = "regression"

        def __init__(self, dim):
            self.raw_dim = dim

        def class_operator(self, class_id):
            from .problems import VALUE

            return VALUE

        def class_data(self, cls):
            return np.asarray(cls.aux["targets"], dtype=np.float64)

    def __init__(self, spec, inputs, targets, weight=None):
        inputs = np.asarray(inputs, dtype=np.float64)
        if inputs.ndim == 1:
            inputs = inputs[:, None]
        targets = np.asarray(targets, dtype=np.float64).reshape(-1)
        if inputs.shape[0] != targets.shape[0]:
            raise DimensionError("inputs and targets disagree on sample count")
        if weight is None:
            weight = 1.0 / np.sqrt(inputs.shape[0])
        colloc = CollocationSet(
            [CollocationClass(INTERIOR, inputs, float(weight), {"targets": targets})]
        )
        super().__init__(self._RegressionProblem(inputs.shape[1]), spec, colloc)

    def rebind(self, collocation):
        cls = collocation.classes[0]
        return RegressionResidualMap(self.spec, cls.points, cls.aux["targets"], cls.weight)


# -- ic_shift output transform (reference model.py:181-277) ------------------------------------


def _is_ic_shift(problem) -> bool:
    tr = getattr(problem, "transform", None)
    return tr is not None and getattr(tr, "kind", "identity") == "ic_shift"


class _IcShiftPart:
    """One half of an ic_shift problem as a plain device problem.

    u(t, x) = phi(t, x) - phi(0, x) + q0(x) (model.py:237-277), so for a linear class
    operator L the residual splits as r = r_A + r_B with
      A: L phi at the points, data f - L q0 (q0's derivatives by host 2-jets);
      B: -L' phi at the points moved to t = 0, data 0, where L' drops every
         time-derivative term (the reference's shift is constant along t,
         model.py:270-272).
    """

    def __init__(self, base, shifted: bool):
        self.base = base
        self.shifted = shifted
        self.name = f"{getattr(base, 'name', 'problem')}:{'shift' if shifted else 'base'}"
        self.raw_dim = base.raw_dim
        self.input_dim = getattr(base, "input_dim", base.raw_dim)
        if hasattr(base, "input_channels"):
            self.input_channels = base.input_channels
        if hasattr(base, "point_grad_dims") or hasattr(base, "point_coefs"):
            raise DomainError("ic_shift with per-point derivative sets is not supported")

    def class_operator(self, class_id):
        from .problems import ClassOperator

        op = self.base.class_operator(class_id)
        if getattr(op, "c3", 0.0):
            raise DomainError("ic_shift needs a linear class operator (u^3 term present)")
        if not self.shifted:
            return op
        keep = [g for g, j in enumerate(op.grad_dims) if j != 0]
        return ClassOperator(cu=-op.cu, grad_dims=tuple(op.grad_dims[g] for g in keep),
                             cg=tuple(-op.cg[g] for g in keep),
                             lap_dims=tuple(j for j in op.lap_dims if j != 0), cl=-op.cl)

    def class_data(self, cls):
        if self.shifted:
            return np.zeros(cls.count)
        from .model import jet_value, point_columns

        op = self.base.class_operator(cls.class_id)
        q0 = self.base.transform.q0
        pts = cls.points
        n = pts.shape[0]
        lq = op.cu * jet_value(q0(point_columns(pts)), n).v
        jets = {j: jet_value(q0(point_columns(pts, j)), n)
                for j in set(op.grad_dims) | set(op.lap_dims)}
        for g, j in enumerate(op.grad_dims):
            lq = lq + op.cg[g] * jets[j].d1
        if op.lap_dims:
            lq = lq + op.cl * sum(jets[j].d2 for j in op.lap_dims)
        return np.asarray(self.base.class_data(cls), dtype=np.float64) - lq


class IcShiftResidualMap(ResidualMap):
    """PINN residual map of a problem with the ic_shift output transform
    (model.py:181-277): two device maps (`_IcShiftPart`) whose residuals, Jacobian
    rows and second directional derivatives add; J is materialised (J = J_A + J_B)
    and the Gram is the SYRK over it.  `PinnResidualMap(problem, ...)` returns this
    map for such problems, so callers construct it exactly as the reference does."""

    graph_capable = False  # candidates' losses need per-candidate residual vectors
    gram_mode = "materialized"

    def __init__(self, problem, spec, collocation: CollocationSet, col_range=None):
        from .model import MlpSpec

        if not isinstance(spec, MlpSpec):
            raise DimensionError("PinnResidualMap needs an MlpSpec")
        if col_range is not None and tuple(col_range) != (0, spec.layout().size):
            raise DomainError("ic_shift maps are not column-sharded")
        self.problem = problem
        self.spec = spec
        self.layout = spec.layout()
        self.collocation = collocation
        self.col_range = (0, self.layout.size)
        shifted = []
        for c in collocation.classes:
            p0 = np.array(c.points, dtype=np.float64, copy=True)
            p0[:, 0] = 0.0
            shifted.append(CollocationClass(c.class_id, p0, c.weight, dict(c.aux)))
        self.A = PinnResidualMap(_IcShiftPart(problem, False), spec, collocation)
        self.B = PinnResidualMap(_IcShiftPart(problem, True), spec, CollocationSet(shifted))
        for part in (self.A, self.B):
            part.gram_mode = "materialized"
        self._cache = None
        self._J = None

    def rebind(self, collocation):
        return IcShiftResidualMap(self.problem, self.spec, collocation)

    def jfree(self) -> bool:
        return False

    def jfree_pcg(self) -> bool:
        return False

    def use_factored_gram(self) -> bool:
        return False

    def _key(self, th):
        return (th.data_ptr(), th._version, id(self.collocation))

    def linearize_t(self, theta):
        import torch

        from . import kernels as K

        th = self._theta_t(theta)
        key = self._key(th)
        if self._cache is not None and self._cache[0] == key:
            return self._cache[1], self._cache[2]
        rA, JA = self.A.linearize_t(th)
        rB, JB = self.B.linearize_t(th)
        if self._J is None or self._J.shape != JA.shape:
            self._J = torch.empty_like(JA)
        r = K.axpby(1.0, rA, 1.0, rB)
        K.axpby(1.0, JA, 1.0, JB, out=self._J)
        self._cache = (key, r, self._J, th)
        return r, self._J

    def residuals_t(self, theta):
        from . import kernels as K

        th = self._theta_t(theta)
        if self._cache is not None and self._cache[0] == self._key(th):
            return self._cache[1]
        return K.axpby(1.0, self.A.residuals_t(th), 1.0, self.B.residuals_t(th))

    def fvv_t(self, theta, v_t):
        from . import kernels as K

        th = self._theta_t(theta)
        return K.axpby(1.0, self.A.fvv_t(th, v_t), 1.0, self.B.fvv_t(th, v_t))

    def loss_many_t(self, cands_t):
        import torch

        from . import kernels as K

        C = cands_t.shape[0]
        out = torch.empty(C, dtype=torch.float64, device=cands_t.device)
        for c in range(C):
            th = cands_t[c]
            r = K.axpby(1.0, self.A.residuals_t(th), 1.0, self.B.residuals_t(th))
            K.dot(r, r, out=out[c:c + 1])
        return K.axpby(0.5, out)
