"""Torch-tensor wrappers over the C ABI (one function per entry point).

Tensors are float64 CUDA tensors owned by the caller; each call runs on the
current torch stream.  Workspaces are cached per (device, size class) so
steady-state steps do not allocate.
"""

from __future__ import annotations

import contextlib
import ctypes

import torch

from . import _lib
from ._lib import c_int, c_size, call, ctx, ptr, stream_handle
from .errors import DimensionError

F64 = torch.float64


def pad_ld(n: int, mult: int = 16) -> int:
    """Leading dimension for J-like matrices: 128-byte row pitch (TMA + coalescing)."""
    return max(mult, (int(n) + mult - 1) // mult * mult)


class Workspace:
    """Grow-only byte arena on the current device."""

    def __init__(self):
        self.buf = None

    def get(self, nbytes: int) -> torch.Tensor:
        nbytes = max(int(nbytes), 256)
        if self.buf is None or self.buf.numel() < nbytes or self.buf.device != torch.device(
            "cuda", torch.cuda.current_device()
        ):
            self.buf = torch.empty(nbytes, dtype=torch.uint8, device="cuda")
        return self.buf


def _ws_tables():
    from ._state import tls

    st = tls()
    return st.ws, st.ws_stack  # per thread: (tag -> Workspace, private graph tables)


@contextlib.contextmanager
def private_workspaces(table: dict):
    """Route workspace() to `table` (a CUDA graph's own buffers, which nothing else
    may grow or free after capture)."""
    stack = _ws_tables()[1]
    stack.append(table)
    try:
        yield
    finally:
        stack.pop()


def workspace(tag: str, nbytes: int) -> torch.Tensor:
    base, stack = _ws_tables()
    table = stack[-1] if stack else base
    ws = table.get(tag)
    if ws is None:
        ws = table[tag] = Workspace()
    return ws.get(nbytes)


def _check2d(A: torch.Tensor, what: str):
    if A.dtype != F64 or not A.is_cuda or A.dim() != 2 or A.stride(1) != 1:
        raise DimensionError(f"{what} must be a row-major float64 CUDA matrix")


# ---------------------------------------------------------------- dense path


def syrk(J: torch.Tensor, ncols: int | None = None, K: torch.Tensor | None = None,
         accumulate: bool = False) -> torch.Tensor:
    """K = J[:, :ncols] J[:, :ncols]^T (full symmetric)."""
    _check2d(J, "J")
    m = J.shape[0]
    ncols = J.shape[1] if ncols is None else int(ncols)
    if K is None:
        K = torch.empty((m, m), dtype=F64, device=J.device)
    nb = c_size()
    call("dngd_syrk_workspace", ctx(), m, ncols, ctypes.byref(nb))
    ws = workspace("syrk", nb.value)
    call("dngd_syrk", ctx(), stream_handle(), ptr(J), m, ncols, J.stride(0), ptr(K), K.stride(0),
         1 if accumulate else 0, ptr(ws), ws.numel())
    return K


def transpose_pad(A: torch.Tensor) -> torch.Tensor:
    """Row-major transpose of a 2-D view into a buffer with a 16-aligned pitch
    (the TMA/GEMM operand layout)."""
    rows, cols = A.shape
    out = torch.zeros((cols, pad_ld(rows)), dtype=F64, device=A.device)
    out[:, :rows].copy_(A.t())
    return out


def shift_copy(K: torch.Tensor, lam: float, L: torch.Tensor) -> torch.Tensor:
    call("dngd_shift_copy", ctx(), stream_handle(), ptr(K), K.shape[0], K.stride(0), float(lam),
         ptr(L), L.stride(0))
    return L


class CholeskyFactor:
    """Lower factor of K + lam I plus the stored diagonal-block inverses."""

    def __init__(self, m: int, device):
        self.m = m
        ld = pad_ld(m, 2)
        self.L = torch.empty((m, ld), dtype=F64, device=device)
        nb = c_size()
        call("dngd_potrf_workspace", ctx(), m, ctypes.byref(nb))
        self.dinv = torch.empty(max(1, (nb.value + 7) // 8), dtype=F64, device=device)
        self.info = torch.zeros(1, dtype=torch.int32, device=device)
        nb = c_size()
        call("dngd_potrs_workspace", ctx(), m, ctypes.byref(nb))
        self.scratch = torch.empty(max(1, (nb.value + 7) // 8), dtype=F64, device=device)

    def factor(self, K: torch.Tensor, lam) -> None:
        """Async: L = chol(lower(K) + lam I); self.info receives the failing column.

        lam is a float, or a (1-element device tensor, multiplier) pair read on
        the device (no host round trip for the damping)."""
        if isinstance(lam, tuple):
            lam_t, mult = lam
            call("dngd_shift_copy_dev", ctx(), stream_handle(), ptr(K), K.shape[0], K.stride(0),
                 ptr(lam_t), float(mult), ptr(self.L), self.L.stride(0))
        else:
            shift_copy(K, lam, self.L)
        call("dngd_potrf", ctx(), stream_handle(), ptr(self.L), self.m, self.L.stride(0),
             ptr(self.dinv), ptr(self.info))

    def solve_(self, b: torch.Tensor) -> torch.Tensor:
        """b <- (L L^T)^{-1} b in place."""
        call("dngd_potrs", ctx(), stream_handle(), ptr(self.L), self.m, self.L.stride(0),
             ptr(self.dinv), ptr(b), ptr(self.scratch))
        return b


def gemv_t(J: torch.Tensor, y: torch.Tensor, ncols: int | None = None, g: torch.Tensor | None = None,
           scale: float = 1.0, out: torch.Tensor | None = None) -> torch.Tensor:
    """out = scale * (J^T y + g)."""
    _check2d(J, "J")
    m = J.shape[0]
    ncols = J.shape[1] if ncols is None else int(ncols)
    if out is None:
        out = torch.empty(ncols, dtype=F64, device=J.device)
    nb = c_size()
    call("dngd_gemv_t_workspace", ctx(), m, ncols, ctypes.byref(nb))
    ws = workspace("gemv_t", nb.value)
    call("dngd_gemv_t", ctx(), stream_handle(), ptr(J), m, ncols, J.stride(0), ptr(y), ptr(g),
         float(scale), ptr(out), ptr(ws), ws.numel())
    return out


def gemv_n(A: torch.Tensor, x: torch.Tensor, ncols: int | None = None, alpha: float = 1.0,
           add: torch.Tensor | None = None, beta: float = 0.0,
           out: torch.Tensor | None = None) -> torch.Tensor:
    """out = alpha * A[:, :ncols] x + beta * add."""
    _check2d(A, "A")
    m = A.shape[0]
    ncols = A.shape[1] if ncols is None else int(ncols)
    if out is None:
        out = torch.empty(m, dtype=F64, device=A.device)
    call("dngd_gemv_n", ctx(), stream_handle(), ptr(A), m, ncols, A.stride(0), ptr(x), float(alpha),
         ptr(add), float(beta), ptr(out))
    return out


def gemm_nt(A: torch.Tensor, B: torch.Tensor, C: torch.Tensor | None = None, K: int | None = None,
            alpha: float = 1.0, beta: float = 0.0, lower: bool = False) -> torch.Tensor:
    """C = alpha * A[:, :K] B[:, :K]^T + beta * C on the FP64 tensor cores."""
    _check2d(A, "A")
    _check2d(B, "B")
    M, N = A.shape[0], B.shape[0]
    K = A.shape[1] if K is None else int(K)
    if C is None:
        C = torch.empty((M, pad_ld(N, 2)), dtype=F64, device=A.device)[:, :N]
    call("dngd_gemm_nt", ctx(), stream_handle(), M, N, K, ptr(A), A.stride(0), 0, ptr(B),
         B.stride(0), 0, ptr(C), C.stride(0), 0, 1, float(alpha), float(beta), 1 if lower else 0)
    return C


def oz_gemm_nt(A: torch.Tensor, B: torch.Tensor, C: torch.Tensor | None = None,
               slices: int = 6) -> torch.Tensor:
    """C = A B^T, emulated FP64 on the int8 tensor cores (Ozaki slices, ozaki.cu)."""
    _check2d(A, "A")
    _check2d(B, "B")
    M, N, K = A.shape[0], B.shape[0], A.shape[1]
    if B.shape[1] != K:
        raise DimensionError("oz_gemm_nt: A and B need the same number of columns")
    if C is None:
        C = torch.empty((M, pad_ld(N, 2)), dtype=F64, device=A.device)[:, :N]
    nb = c_size(0)
    call("dngd_oz_gemm_workspace", ctx(), M, N, K, int(slices), ctypes.byref(nb))
    ws = workspace("oz_gemm", nb.value)
    call("dngd_oz_gemm_nt", ctx(), stream_handle(), M, N, K, ptr(A), A.stride(0), ptr(B),
         B.stride(0), ptr(C), C.stride(0), int(slices), ptr(ws), ws.numel())
    return C


def dot(x: torch.Tensor, y: torch.Tensor, out: torch.Tensor | None = None) -> torch.Tensor:
    if out is None:
        out = torch.empty(1, dtype=F64, device=x.device)
    call("dngd_dot", ctx(), stream_handle(), x.numel(), ptr(x), ptr(y), ptr(out))
    return out


def axpby(a: float, x: torch.Tensor, b: float = 0.0, y: torch.Tensor | None = None,
          out: torch.Tensor | None = None) -> torch.Tensor:
    if out is None:
        out = torch.empty_like(x)
    call("dngd_axpby", ctx(), stream_handle(), x.numel(), float(a), ptr(x), float(b), ptr(y),
         ptr(out))
    return out


def ls_select(losses, etas, rr, info, anyd, reject_if_worse, mult, sel):
    """Device-side line-search selection and accept/reject bookkeeping (see the
    header): sel <- (eta, loss after, status, index); mult updated in place."""
    call("dngd_ls_select", ctx(), stream_handle(), ptr(losses), losses.numel(), ptr(etas), ptr(rr),
         ptr(info), ptr(anyd), int(bool(reject_if_worse)), ptr(mult), ptr(sel))


def ga_combine(v, a, scal, out, anyd):
    """out = v + a/2 if the GA gate (from scal[2:4] = |v|^2, |a|^2) is open, else v;
    anyd (zeroed by the caller) becomes 1 if out has a nonzero entry."""
    call("dngd_ga_combine", ctx(), stream_handle(), v.numel(), ptr(v), ptr(a), ptr(scal), ptr(out),
         ptr(anyd))
    return out


def theta_update(theta, delta, sel, out):
    """out = theta + sel[0] delta when sel[2] == 0 (accepted), else theta."""
    call("dngd_theta_update", ctx(), stream_handle(), theta.numel(), ptr(theta), ptr(delta),
         ptr(sel), ptr(out))
    return out


# ---------------------------------------------------------------- PINN map


def mlp_desc(widths) -> _lib.MlpDesc:
    d = _lib.MlpDesc()
    d.nlayers = len(widths) - 1
    if d.nlayers > _lib.MAX_LAYERS:
        raise DimensionError(f"at most {_lib.MAX_LAYERS} layers are supported")
    for k, w in enumerate(widths):
        d.widths[k] = int(w)
    return d


def pinn_workspace_bytes(mlp, classes_arr, nclass: int, ncand: int) -> int:
    nb = c_size()
    call("dngd_pinn_workspace", ctx(), ctypes.byref(mlp), classes_arr, nclass, ncand,
         ctypes.byref(nb))
    return nb.value


def assemble(mlp, theta, classes_arr, nclass, r, J=None, col_begin=0, col_end=None, ws=None):
    n = sum((mlp.widths[k] + 1) * mlp.widths[k + 1] for k in range(mlp.nlayers))
    col_end = n if col_end is None else col_end
    call("dngd_assemble", ctx(), stream_handle(), ctypes.byref(mlp), ptr(theta), classes_arr, nclass,
         int(col_begin), int(col_end), ptr(r), ptr(J), 0 if J is None else J.stride(0), ptr(ws),
         0 if ws is None else ws.numel())


def gram_factored(mlp, theta, classes_arr, nclass, r, K, ws, part=0, nparts=1):
    """r and K = J J^T from the activations (J never materialised).  With nparts > 1
    only the part-th of nparts equal tile ranges of K is written (tile-sharded Gram)."""
    if nparts == 1:
        call("dngd_gram_factored", ctx(), stream_handle(), ctypes.byref(mlp), ptr(theta),
             classes_arr, nclass, ptr(r), ptr(K), K.stride(0), ptr(ws), ws.numel())
    else:
        call("dngd_gram_factored_part", ctx(), stream_handle(), ctypes.byref(mlp), ptr(theta),
             classes_arr, nclass, ptr(r), ptr(K), K.stride(0), int(part), int(nparts), ptr(ws),
             ws.numel())


def gram_emulation_slices(mlp=None) -> int:
    """Ozaki digit count of the factored Gram's G-space products (0 = FP64 DMMA).
    DNGD_GRAM_SLICES (0, 6 or 7) overrides; by default hidden layers 64 wide or more
    run emulated with 6 balanced base-256 digits (48 bits below each row's maximum, 21
    int8 products per FP64 product; 7 digits = 56 bits, 28 products) and narrower nets
    stay on DMMA (a 32-wide layer is one K-chunk per phase: the TMEM drains would
    dominate)."""
    import os

    env = os.environ.get("DNGD_GRAM_SLICES")
    if env is not None:
        v = int(env)
        if v not in (0, 6, 7):
            raise DimensionError("DNGD_GRAM_SLICES must be 0, 6 or 7")
        return v
    if mlp is None:
        return 6
    hidden = [mlp.widths[k] for k in range(1, mlp.nlayers)]
    return 6 if hidden and max(hidden) >= 64 else 0


def gram_factored_act(mlp, classes_arr, nclass, K, act_ws, part=0, nparts=1, slices=None):
    """K (or part `part` of nparts of its tiles) from the activations in act_ws: the
    G-space products on the int8 tensor cores (Ozaki slices, gram_oz.cuh) unless
    slices == 0, then on the FP64 DMMA pipe (gram_factored.cuh)."""
    auto = slices is None
    slices = gram_emulation_slices(mlp) if auto else int(slices)
    if slices:
        nb = c_size(0)
        lib = _lib.load_library()
        rc = lib.dngd_gram_oz_workspace(ctx(), ctypes.byref(mlp), classes_arr, nclass, slices,
                                        ctypes.byref(nb))
        if rc == _lib.DNGD_ERR_UNSUPPORTED and auto:
            # outside the emulated kernel's shapes (goz_check: input dim, channels per
            # point, layer width): the FP64 DMMA kernel computes the same K
            return gram_factored_act(mlp, classes_arr, nclass, K, act_ws, part, nparts, 0)
        _lib.check(rc, "dngd_gram_oz_workspace")
        ows = workspace("gram_oz", nb.value)
        call("dngd_gram_oz_act", ctx(), stream_handle(), ctypes.byref(mlp), classes_arr, nclass,
             ptr(K), K.stride(0), int(part), int(nparts), slices, ptr(act_ws), act_ws.numel(),
             ptr(ows), ows.numel())
        return
    call("dngd_gram_factored_act", ctx(), stream_handle(), ctypes.byref(mlp), classes_arr, nclass,
         ptr(K), K.stride(0), int(part), int(nparts), ptr(act_ws), act_ws.numel())


def activations(mlp, theta, classes_arr, nclass, r, ws):
    """r and the forward / adjoint activations (no J) into ws."""
    call("dngd_activations", ctx(), stream_handle(), ctypes.byref(mlp), ptr(theta), classes_arr,
         nclass, ptr(r), ptr(ws), ws.numel())


def jt_workspace_bytes(mlp, classes_arr, nclass) -> int:
    nb = c_size()
    call("dngd_jt_workspace", ctx(), ctypes.byref(mlp), classes_arr, nclass, ctypes.byref(nb))
    return nb.value


def jt_factored(mlp, classes_arr, nclass, w, scale, out, act_ws, scratch):
    """out = scale * J^T w from the activations in act_ws (no J)."""
    call("dngd_jt_factored", ctx(), stream_handle(), ctypes.byref(mlp), classes_arr, nclass, ptr(w),
         float(scale), ptr(out), ptr(act_ws), act_ws.numel(), ptr(scratch), scratch.numel())


def jt_factored_range(mlp, classes_arr, nclass, w, scale, out, c0, c1, act_ws, scratch):
    """out = scale * (J^T w)[c0:c1] from the activations in act_ws (no J)."""
    call("dngd_jt_factored_range", ctx(), stream_handle(), ctypes.byref(mlp), classes_arr, nclass,
         ptr(w), float(scale), ptr(out), int(c0), int(c1), ptr(act_ws), act_ws.numel(),
         ptr(scratch), scratch.numel())


def fvv(mlp, theta, v, classes_arr, nclass, out, ws, act_ws=None):
    """f_vv; act_ws (activations at the same theta) lets the large-din input layer
    reuse x W0 instead of recomputing it."""
    if act_ws is None:
        call("dngd_fvv", ctx(), stream_handle(), ctypes.byref(mlp), ptr(theta), ptr(v),
             classes_arr, nclass, ptr(out), ptr(ws), ws.numel())
    else:
        call("dngd_fvv_act", ctx(), stream_handle(), ctypes.byref(mlp), ptr(theta), ptr(v),
             classes_arr, nclass, ptr(out), ptr(ws), ws.numel(), ptr(act_ws), act_ws.numel())


def gram_factored_cols(mlp, classes_arr, nclass, landmarks, Kc, act_ws):
    """Kc (m x ell) = K[:, landmarks] from the activations in act_ws (no J)."""
    import numpy as _np

    lm = _np.ascontiguousarray(landmarks, dtype=_np.int64)
    nb = c_size()
    call("dngd_gram_cols_workspace", ctx(), ctypes.byref(mlp), classes_arr, nclass, int(lm.size),
         ctypes.byref(nb))
    scratch = workspace("gram_cols", nb.value)
    call("dngd_gram_factored_cols", ctx(), stream_handle(), ctypes.byref(mlp), classes_arr,
         nclass, lm.ctypes.data_as(ctypes.c_void_p), int(lm.size), ptr(Kc), Kc.stride(0),
         ptr(act_ws), act_ws.numel(), ptr(scratch), scratch.numel())


def jvp_factored(mlp, theta, v, classes_arr, nclass, out, ws):
    """out = J v from forward tangents (no J)."""
    call("dngd_jvp_factored", ctx(), stream_handle(), ctypes.byref(mlp), ptr(theta), ptr(v),
         classes_arr, nclass, ptr(out), ptr(ws), ws.numel())


def loss_many(mlp, theta, delta, etas, ncand, classes_arr, nclass, out, ws, act_ws=None):
    if act_ws is None:
        call("dngd_loss_many", ctx(), stream_handle(), ctypes.byref(mlp), ptr(theta), ptr(delta),
             ptr(etas), int(ncand), classes_arr, nclass, ptr(out), ptr(ws), ws.numel())
    else:
        call("dngd_loss_many_act", ctx(), stream_handle(), ctypes.byref(mlp), ptr(theta),
             ptr(delta), ptr(etas), int(ncand), classes_arr, nclass, ptr(out), ptr(ws), ws.numel(),
             ptr(act_ws), act_ws.numel())


def nonfinite_report(x: torch.Tensor, class_ends):
    """(class index, point index) of the first non-finite entry of x, or None
    (dngd_nonfinite_report: a device scan, one synchronisation)."""
    import numpy as _np

    ends = _np.ascontiguousarray(class_ends, dtype=_np.int64)
    cls, pt = c_int(-1), ctypes.c_int64(-1)
    rc = _lib.load_library().dngd_nonfinite_report(
        ctx(), stream_handle(), ptr(x), x.numel(), ends.ctypes.data_as(ctypes.c_void_p),
        len(ends), ctypes.byref(cls), ctypes.byref(pt))
    if rc == _lib.DNGD_OK:
        return None
    if rc != _lib.DNGD_ERR_NONFINITE:
        _lib.check(rc, "dngd_nonfinite_report")
    return cls.value, pt.value


# ---------------------------------------------------------------- Nystrom-PCG numerics


def syev_jacobi(A: torch.Tensor, n: int | None = None):
    """(w, V, sweeps) of the symmetric n x n matrix A (device): A = V diag(w) V^T by
    the library's Jacobi eigensolver; eigenpairs unsorted."""
    _check2d(A, "A")
    n = A.shape[0] if n is None else int(n)
    nb = c_size()
    call("dngd_syev_workspace", ctx(), n, ctypes.byref(nb))
    ws = workspace("syev", nb.value)
    w = torch.empty(n, dtype=F64, device=A.device)
    V = torch.empty((n, pad_ld(n, 2)), dtype=F64, device=A.device)[:, :n]
    sweeps = torch.zeros(1, dtype=torch.int32, device=A.device)
    call("dngd_syev_jacobi", ctx(), stream_handle(), ptr(A), n, A.stride(0), ptr(w), ptr(V),
         V.stride(0), ptr(sweeps), ptr(ws), ws.numel())
    return w, V, sweeps


def nystrom_scale(V, w, floor_rel, Wt, Qst, rank_dev):
    l = w.numel()
    call("dngd_nystrom_scale", ctx(), stream_handle(), ptr(V), V.stride(0), ptr(w), l,
         float(floor_rel), ptr(Wt), Wt.stride(0), ptr(Qst), Qst.stride(0), ptr(rank_dev))


def pivoted_cholesky(Kmat, l, tol, Lt, k_dev):
    """Lt (k x l) with K ~ L L^T (diagonal pivoting, stop at tol * max diag)."""
    ws = workspace("pivchol", 12 * l + 64)
    call("dngd_pivoted_cholesky", ctx(), stream_handle(), ptr(Kmat), int(l), Kmat.stride(0),
         float(tol), Lt.shape[0], ptr(Lt), Lt.stride(0), ptr(ws), ws.numel(), ptr(k_dev))


def nystrom_from_chol(W, lam, k, Lt, l, floor_rel, Wt, Qst, rank_dev):
    call("dngd_nystrom_from_chol", ctx(), stream_handle(), ptr(W), W.stride(0), ptr(lam), int(k),
         ptr(Lt), Lt.stride(0), int(l), float(floor_rel), ptr(Wt), Wt.stride(0), ptr(Qst),
         Qst.stride(0), ptr(rank_dev))


def nystrom_scatter(Qst, landmarks_dev, Mt):
    """Mt[r, landmarks[i]] = Qst[r, i] for every row r of Mt."""
    call("dngd_nystrom_scatter", ctx(), stream_handle(), ptr(Qst), Qst.stride(0), Mt.shape[0],
         landmarks_dev.numel(), ptr(landmarks_dev), ptr(Mt), Mt.stride(0))


def cg_init(state, tol, max_iters):
    call("dngd_cg_init", ctx(), stream_handle(), ptr(state), float(tol), int(max_iters))


def cg_after_pap(state, y, r, p, Ap):
    call("dngd_cg_after_pap", ctx(), stream_handle(), ptr(state), y.numel(), ptr(y), ptr(r),
         ptr(p), ptr(Ap))


def cg_after_r(state, y, ybest, flag):
    call("dngd_cg_after_r", ctx(), stream_handle(), ptr(state), y.numel(), ptr(y), ptr(ybest),
         ptr(flag))


def cg_update_p(state, p, z, flag, cond):
    call("dngd_cg_update_p", ctx(), stream_handle(), ptr(state), p.numel(), ptr(p), ptr(z),
         ptr(flag), ctypes.c_uint64(int(cond)))


def cg_finish(state, y, ybest, radd=None):
    call("dngd_cg_finish", ctx(), stream_handle(), ptr(state), y.numel(), ptr(y), ptr(ybest),
         ptr(radd))


def axmy(c, v, u, out):
    """out = c (v - u)."""
    call("dngd_axmy", ctx(), stream_handle(), v.numel(), float(c), ptr(v), ptr(u), ptr(out))
    return out


class LoopGraph:
    """A CUDA graph with one WHILE conditional node whose body is captured from the
    library calls made inside `capture()` (see dngd_loop_graph_*)."""

    def __init__(self):
        h = ctypes.c_void_p()
        cond = ctypes.c_uint64()
        call("dngd_loop_graph_create", ctx(), ctypes.byref(h), ctypes.byref(cond))
        self.handle, self.cond = h, cond.value
        self._ctx = ctx()

    @contextlib.contextmanager
    def capture(self, stream):
        """Body capture on `stream` (a torch.cuda.Stream made current meanwhile).
        Nothing inside may allocate device memory through torch."""
        with torch.cuda.stream(stream):
            call("dngd_loop_graph_begin", ctx(), self.handle, ctypes.c_void_p(stream.cuda_stream))
            try:
                yield
            finally:
                call("dngd_loop_graph_end", ctx(), self.handle, ctypes.c_void_p(stream.cuda_stream))

    def launch(self):
        call("dngd_loop_graph_launch", ctx(), self.handle, stream_handle())

    def __del__(self):
        try:
            if self.handle:
                _lib.load_library().dngd_loop_graph_destroy(self._ctx, self.handle)
        except Exception:
            pass
