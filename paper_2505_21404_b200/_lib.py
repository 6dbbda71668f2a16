"""ctypes binding of libdngd_b200.so (the C ABI in include/dngd_b200.h).

There is no CPU fallback: importing the product on a machine without the
built library or without an sm_100 device raises immediately.
"""

from __future__ import annotations

import ctypes
import os
import threading

import torch

from .errors import DimensionError, DngdError, DomainError, FactorizationError, NonFiniteError

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "libdngd_b200.so")

DNGD_OK = 0
DNGD_ERR_DIMENSION = 1
DNGD_ERR_DOMAIN = 2
DNGD_ERR_NOT_PD = 3
DNGD_ERR_NONFINITE = 4
DNGD_ERR_CUDA = 5
DNGD_ERR_UNSUPPORTED = 6

MAX_LAYERS = 8
MAX_CLASSES = 4
MAX_GRAD = 12

c_i64 = ctypes.c_int64
c_dbl = ctypes.c_double
c_int = ctypes.c_int
c_vp = ctypes.c_void_p
c_size = ctypes.c_size_t


class MlpDesc(ctypes.Structure):
    _fields_ = [("nlayers", c_int), ("widths", c_int * (MAX_LAYERS + 1))]


class ClassDesc(ctypes.Structure):
    _fields_ = [
        ("count", c_i64),
        ("ngrad", c_int),
        ("nlap", c_int),
        ("grad_dims", c_int * MAX_GRAD),
        ("lap_grad", c_int * MAX_GRAD),
        ("cg", c_dbl * MAX_GRAD),
        ("cu", c_dbl),
        ("cl", c_dbl),
        ("weight", c_dbl),
        ("points", c_vp),
        ("f", c_vp),
        ("c3", c_dbl),
        ("inputs", c_vp),
        ("grad_idx", c_vp),
        ("coefs", c_vp),
    ]


_SIGS = {
    "dngd_version": ([], c_int),
    "dngd_ctx_create": ([c_int, ctypes.POINTER(c_vp)], c_int),
    "dngd_ctx_destroy": ([c_vp], c_int),
    "dngd_ctx_last_error": ([c_vp], ctypes.c_char_p),
    "dngd_syrk_workspace": ([c_vp, c_i64, c_i64, ctypes.POINTER(c_size)], c_int),
    "dngd_syrk": ([c_vp, c_vp, c_vp, c_i64, c_i64, c_i64, c_vp, c_i64, c_int, c_vp, c_size], c_int),
    "dngd_potrf_workspace": ([c_vp, c_i64, ctypes.POINTER(c_size)], c_int),
    "dngd_shift_copy": ([c_vp, c_vp, c_vp, c_i64, c_i64, c_dbl, c_vp, c_i64], c_int),
    "dngd_shift_copy_dev": ([c_vp, c_vp, c_vp, c_i64, c_i64, c_vp, c_dbl, c_vp, c_i64], c_int),
    "dngd_potrf": ([c_vp, c_vp, c_vp, c_i64, c_i64, c_vp, c_vp], c_int),
    "dngd_potrs_workspace": ([c_vp, c_i64, ctypes.POINTER(c_size)], c_int),
    "dngd_potrs": ([c_vp, c_vp, c_vp, c_i64, c_i64, c_vp, c_vp, c_vp], c_int),
    "dngd_gemv_t_workspace": ([c_vp, c_i64, c_i64, ctypes.POINTER(c_size)], c_int),
    "dngd_gemv_t": ([c_vp, c_vp, c_vp, c_i64, c_i64, c_i64, c_vp, c_vp, c_dbl, c_vp, c_vp, c_size], c_int),
    "dngd_gemv_n": ([c_vp, c_vp, c_vp, c_i64, c_i64, c_i64, c_vp, c_dbl, c_vp, c_dbl, c_vp], c_int),
    "dngd_gemm_nt": ([c_vp, c_vp, c_i64, c_i64, c_i64, c_vp, c_i64, c_i64, c_vp, c_i64, c_i64,
                      c_vp, c_i64, c_i64, c_int, c_dbl, c_dbl, c_int], c_int),
    "dngd_oz_gemm_workspace": ([c_vp, c_i64, c_i64, c_i64, c_int, ctypes.POINTER(c_size)], c_int),
    "dngd_oz_gemm_nt": ([c_vp, c_vp, c_i64, c_i64, c_i64, c_vp, c_i64, c_vp, c_i64, c_vp, c_i64,
                         c_int, c_vp, c_size], c_int),
    "dngd_dot": ([c_vp, c_vp, c_i64, c_vp, c_vp, c_vp], c_int),
    "dngd_axpby": ([c_vp, c_vp, c_i64, c_dbl, c_vp, c_dbl, c_vp, c_vp], c_int),
    "dngd_ls_select": ([c_vp, c_vp, c_vp, c_int, c_vp, c_vp, c_vp, c_vp, c_int, c_vp, c_vp], c_int),
    "dngd_theta_update": ([c_vp, c_vp, c_i64, c_vp, c_vp, c_vp, c_vp], c_int),
    "dngd_ga_combine": ([c_vp, c_vp, c_i64, c_vp, c_vp, c_vp, c_vp, c_vp], c_int),
    "dngd_pinn_workspace": ([c_vp, ctypes.POINTER(MlpDesc), ctypes.POINTER(ClassDesc), c_int, c_int,
                             ctypes.POINTER(c_size)], c_int),
    "dngd_assemble": ([c_vp, c_vp, ctypes.POINTER(MlpDesc), c_vp, ctypes.POINTER(ClassDesc), c_int,
                       c_i64, c_i64, c_vp, c_vp, c_i64, c_vp, c_size], c_int),
    "dngd_gram_factored": ([c_vp, c_vp, ctypes.POINTER(MlpDesc), c_vp, ctypes.POINTER(ClassDesc),
                            c_int, c_vp, c_vp, c_i64, c_vp, c_size], c_int),
    "dngd_gram_factored_part": ([c_vp, c_vp, ctypes.POINTER(MlpDesc), c_vp,
                                 ctypes.POINTER(ClassDesc), c_int, c_vp, c_vp, c_i64, c_int,
                                 c_int, c_vp, c_size], c_int),
    "dngd_gram_factored_act": ([c_vp, c_vp, ctypes.POINTER(MlpDesc), ctypes.POINTER(ClassDesc),
                                c_int, c_vp, c_i64, c_int, c_int, c_vp, c_size], c_int),
    "dngd_gram_oz_workspace": ([c_vp, ctypes.POINTER(MlpDesc), ctypes.POINTER(ClassDesc), c_int,
                                c_int, ctypes.POINTER(c_size)], c_int),
    "dngd_gram_oz_act": ([c_vp, c_vp, ctypes.POINTER(MlpDesc), ctypes.POINTER(ClassDesc), c_int,
                          c_vp, c_i64, c_int, c_int, c_int, c_vp, c_size, c_vp, c_size], c_int),
    "dngd_activations": ([c_vp, c_vp, ctypes.POINTER(MlpDesc), c_vp, ctypes.POINTER(ClassDesc),
                          c_int, c_vp, c_vp, c_size], c_int),
    "dngd_jt_workspace": ([c_vp, ctypes.POINTER(MlpDesc), ctypes.POINTER(ClassDesc), c_int,
                           ctypes.POINTER(c_size)], c_int),
    "dngd_jt_factored": ([c_vp, c_vp, ctypes.POINTER(MlpDesc), ctypes.POINTER(ClassDesc), c_int,
                          c_vp, c_dbl, c_vp, c_vp, c_size, c_vp, c_size], c_int),
    "dngd_jt_factored_range": ([c_vp, c_vp, ctypes.POINTER(MlpDesc), ctypes.POINTER(ClassDesc),
                                c_int, c_vp, c_dbl, c_vp, c_i64, c_i64, c_vp, c_size, c_vp,
                                c_size], c_int),
    "dngd_fvv": ([c_vp, c_vp, ctypes.POINTER(MlpDesc), c_vp, c_vp, ctypes.POINTER(ClassDesc), c_int,
                  c_vp, c_vp, c_size], c_int),
    "dngd_gram_cols_workspace": ([c_vp, ctypes.POINTER(MlpDesc), ctypes.POINTER(ClassDesc), c_int,
                                  c_int, ctypes.POINTER(c_size)], c_int),
    "dngd_gram_factored_cols": ([c_vp, c_vp, ctypes.POINTER(MlpDesc), ctypes.POINTER(ClassDesc),
                                 c_int, c_vp, c_int, c_vp, c_i64, c_vp, c_size, c_vp, c_size],
                                c_int),
    "dngd_jvp_factored": ([c_vp, c_vp, ctypes.POINTER(MlpDesc), c_vp, c_vp,
                           ctypes.POINTER(ClassDesc), c_int, c_vp, c_vp, c_size], c_int),
    "dngd_loss_many": ([c_vp, c_vp, ctypes.POINTER(MlpDesc), c_vp, c_vp, c_vp, c_int,
                        ctypes.POINTER(ClassDesc), c_int, c_vp, c_vp, c_size], c_int),
    "dngd_fvv_act": ([c_vp, c_vp, ctypes.POINTER(MlpDesc), c_vp, c_vp, ctypes.POINTER(ClassDesc),
                      c_int, c_vp, c_vp, c_size, c_vp, c_size], c_int),
    "dngd_loss_many_act": ([c_vp, c_vp, ctypes.POINTER(MlpDesc), c_vp, c_vp, c_vp, c_int,
                            ctypes.POINTER(ClassDesc), c_int, c_vp, c_vp, c_size, c_vp, c_size],
                           c_int),
    "dngd_nonfinite_report": ([c_vp, c_vp, c_vp, c_i64, c_vp, c_int, ctypes.POINTER(c_int),
                               ctypes.POINTER(c_i64)], c_int),
    "dngd_syev_workspace": ([c_vp, c_i64, ctypes.POINTER(c_size)], c_int),
    "dngd_syev_jacobi": ([c_vp, c_vp, c_vp, c_i64, c_i64, c_vp, c_vp, c_i64, c_vp, c_vp, c_size],
                         c_int),
    "dngd_nystrom_scale": ([c_vp, c_vp, c_vp, c_i64, c_vp, c_int, c_dbl, c_vp, c_i64, c_vp, c_i64,
                            c_vp], c_int),
    "dngd_pivoted_cholesky": ([c_vp, c_vp, c_vp, c_i64, c_i64, c_dbl, c_int, c_vp, c_i64, c_vp,
                               c_size, c_vp], c_int),
    "dngd_nystrom_from_chol": ([c_vp, c_vp, c_vp, c_i64, c_vp, c_int, c_vp, c_i64, c_int, c_dbl,
                                c_vp, c_i64, c_vp, c_i64, c_vp], c_int),
    "dngd_nystrom_scatter": ([c_vp, c_vp, c_vp, c_i64, c_int, c_int, c_vp, c_vp, c_i64], c_int),
    "dngd_cg_init": ([c_vp, c_vp, c_vp, c_dbl, c_int], c_int),
    "dngd_cg_after_pap": ([c_vp, c_vp, c_vp, c_i64, c_vp, c_vp, c_vp, c_vp], c_int),
    "dngd_cg_after_r": ([c_vp, c_vp, c_vp, c_i64, c_vp, c_vp, c_vp], c_int),
    "dngd_cg_update_p": ([c_vp, c_vp, c_vp, c_i64, c_vp, c_vp, c_vp, ctypes.c_uint64], c_int),
    "dngd_cg_finish": ([c_vp, c_vp, c_vp, c_i64, c_vp, c_vp, c_vp], c_int),
    "dngd_axmy": ([c_vp, c_vp, c_i64, c_dbl, c_vp, c_vp, c_vp], c_int),
    "dngd_loop_graph_create": ([c_vp, ctypes.POINTER(c_vp), ctypes.POINTER(ctypes.c_uint64)], c_int),
    "dngd_loop_graph_begin": ([c_vp, c_vp, c_vp], c_int),
    "dngd_loop_graph_end": ([c_vp, c_vp, c_vp], c_int),
    "dngd_loop_graph_launch": ([c_vp, c_vp, c_vp], c_int),
    "dngd_loop_graph_destroy": ([c_vp, c_vp], c_int),
}

EXPORTED = tuple(_SIGS)

_lib = None
_lock = threading.Lock()
_tls = threading.local()


def load_library(path: str = LIB_PATH) -> ctypes.CDLL:
    """Load the shared library (no device needed); raises if it was never built."""
    global _lib
    with _lock:
        if _lib is None:
            if not os.path.exists(path):
                raise DngdError(
                    f"{path} is missing: build it with paper_2505_21404_b200._build.build_library() "
                    "(there is no CPU fallback)"
                )
            lib = ctypes.CDLL(path)
            for name, (args, res) in _SIGS.items():
                fn = getattr(lib, name)
                fn.argtypes = args
                fn.restype = res
            _lib = lib
    return _lib


class _Ctx:
    def __init__(self, device: int):
        lib = load_library()
        h = c_vp()
        rc = lib.dngd_ctx_create(device, ctypes.byref(h))
        if rc != DNGD_OK:
            raise DngdError(f"dngd_ctx_create(device={device}) failed with status {rc}: "
                            "an sm_100 (B200) CUDA device is required")
        self.handle = h
        self.device = device

    def __del__(self):
        try:
            if _lib is not None and self.handle:
                _lib.dngd_ctx_destroy(self.handle)
        except Exception:
            pass


def require_cuda() -> torch.device:
    if not torch.cuda.is_available():
        raise DngdError("paper_2505_21404_b200 needs a CUDA device (B200, sm_100a); "
                        "there is no CPU fallback")
    return torch.device("cuda", torch.cuda.current_device())


def ctx() -> ctypes.c_void_p:
    """Per-thread, per-device context (the ABI is reentrant; state lives here)."""
    dev = require_cuda().index
    cache = getattr(_tls, "ctx", None)
    if cache is None:
        cache = _tls.ctx = {}
    c = cache.get(dev)
    if c is None:
        c = cache[dev] = _Ctx(dev)
    return c.handle


def stream_handle() -> ctypes.c_void_p:
    return c_vp(torch.cuda.current_stream().cuda_stream)


def check(rc: int, what: str) -> None:
    if rc == DNGD_OK:
        return
    msg = _lib.dngd_ctx_last_error(ctx()).decode(errors="replace")
    text = f"{what}: {msg}" if msg else f"{what} failed (status {rc})"
    if rc == DNGD_ERR_DIMENSION:
        raise DimensionError(text)
    if rc == DNGD_ERR_DOMAIN:
        raise DomainError(text)
    if rc == DNGD_ERR_NOT_PD:
        raise FactorizationError(text)
    if rc == DNGD_ERR_NONFINITE:
        raise NonFiniteError(text)
    raise DngdError(text)


def call(name: str, *args) -> None:
    lib = load_library()
    check(getattr(lib, name)(*args), name)


def ptr(t) -> ctypes.c_void_p:
    if t is None:
        return c_vp(None)
    return c_vp(t.data_ptr())
