"""ctypes binding of the C ABI in include/brsvd.h (libbrsvd: ``_brsvd.so``).

The product path has no CPU fallback: if the shared library is missing or no
CUDA device is visible, every entry point raises ``BackendUnavailable``.
Build the library with ``python -m paper_1706_07191_b200.build`` (or
``__graft_entry__.build()``).
"""

import ctypes
import os
import threading

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "_brsvd.so")

OK, ERR_CONFIG, ERR_SHAPE, ERR_BUDGET, ERR_OVERFLOW, ERR_CUDA, ERR_NCCL, ERR_ARG = range(8)
F64, F32 = 1, 2
COL_MAJOR, ROW_MAJOR = 0, 1
DEVICE, HOST = 0, 1

EXPORTED = (
    "brsvd_version", "brsvd_last_error", "brsvd_ctx_create", "brsvd_ctx_set_stream",
    "brsvd_ctx_destroy", "brsvd_rsvd", "brsvd_tsqr", "brsvd_small_svd",
    "brsvd_gaussian", "brsvd_profile_begin", "brsvd_profile_end",
    "brsvd_spectral_norm", "brsvd_ialm", "brsvd_sketch_product", "brsvd_gram",
    "brsvd_chol_basis", "brsvd_apply", "brsvd_normalize", "brsvd_colmax",
    "brsvd_scale_cols", "brsvd_rsvd_stream", "brsvd_residual", "brsvd_rsvd_blocked",
    "brsvd_rsvd_stream_blocked", "brsvd_ialm_blocked", "brsvd_sketch_product_scaled",
    "brsvd_absmax", "brsvd_range_finder", "brsvd_colmax_entries", "brsvd_stream_rows_pass",
    "brsvd_normalize_f64", "brsvd_ialm_stream", "brsvd_spectral_norm_start",
    "brsvd_nccl_unique_id", "brsvd_ctx_attach_nccl", "brsvd_allreduce", "brsvd_allgather",
    "brsvd_normalize_t", "brsvd_unnormalised_peak",
)


class BackendUnavailable(RuntimeError):
    """The CUDA extension is not built or no GPU is visible."""


class BrsvdStats(ctypes.Structure):
    _fields_ = [
        ("words_read", ctypes.c_int64),
        ("block_reads", ctypes.c_int64),
        ("passes_num", ctypes.c_int64),
        ("passes_den", ctypes.c_int64),
        ("flop_estimate", ctypes.c_int64),
        ("detected_rank", ctypes.c_int32),
        ("core_rank", ctypes.c_int32),
        ("max_abs_y0", ctypes.c_double),
        ("log10_peak_est", ctypes.c_double),
        ("overflow", ctypes.c_int32),
        ("reserved", ctypes.c_int32),
        ("seconds_sketch", ctypes.c_double),
        ("seconds_orthonormalize", ctypes.c_double),
        ("seconds_form_core", ctypes.c_double),
        ("seconds_svd", ctypes.c_double),
    ]


class BrsvdProfile(ctypes.Structure):
    _fields_ = [
        ("big_launches", ctypes.c_int64),
        ("big_ms", ctypes.c_double),
        ("big_flops", ctypes.c_double),
        ("big_bytes", ctypes.c_double),
        ("gpu_launches", ctypes.c_int64),
    ]


_lib = None
_lib_lock = threading.Lock()
_tls = threading.local()


def _declare(lib):
    vp, i64, i32, u64, c_int = (ctypes.c_void_p, ctypes.c_int64, ctypes.c_int32,
                                ctypes.c_uint64, ctypes.c_int)
    lib.brsvd_version.restype = c_int
    lib.brsvd_last_error.restype = ctypes.c_char_p
    lib.brsvd_ctx_create.argtypes = [c_int, vp, ctypes.POINTER(vp)]
    lib.brsvd_ctx_set_stream.argtypes = [vp, vp]
    lib.brsvd_ctx_destroy.argtypes = [vp]
    lib.brsvd_rsvd.argtypes = [vp, vp, i64, i64, i64, c_int, c_int, c_int, c_int, c_int,
                               c_int, vp, c_int, u64, vp, vp, vp, c_int,
                               ctypes.POINTER(BrsvdStats)]
    lib.brsvd_rsvd_blocked.argtypes = [vp, vp, i64, i64, i64, c_int, c_int, c_int, c_int,
                                       c_int, c_int, vp, c_int, u64, vp, c_int, vp, vp, vp,
                                       c_int, ctypes.POINTER(BrsvdStats)]
    lib.brsvd_range_finder.argtypes = [vp, vp, i64, i64, i64, c_int, c_int, c_int, c_int,
                                       c_int, c_int, vp, c_int, u64, vp, c_int, vp, c_int,
                                       ctypes.POINTER(BrsvdStats)]
    lib.brsvd_tsqr.argtypes = [vp, vp, i64, i64, i64, c_int, c_int, vp, vp,
                               ctypes.POINTER(i32)]
    lib.brsvd_small_svd.argtypes = [vp, vp, i64, i64, i64, c_int, c_int, vp, vp, vp,
                                    ctypes.POINTER(i32)]
    lib.brsvd_gaussian.argtypes = [vp, vp, i64, i64, i64, c_int, u64, u64, i64]
    dbl = ctypes.c_double
    lib.brsvd_spectral_norm.argtypes = [vp, vp, i64, i64, i64, c_int, c_int, c_int, u64,
                                        dbl, c_int, ctypes.POINTER(dbl),
                                        ctypes.POINTER(i32)]
    lib.brsvd_spectral_norm_start.argtypes = [vp, vp, i64, i64, i64, c_int, c_int, c_int, u64,
                                              vp, dbl, c_int, ctypes.POINTER(dbl),
                                              ctypes.POINTER(i32)]
    lib.brsvd_nccl_unique_id.argtypes = [ctypes.c_char_p]
    lib.brsvd_ctx_attach_nccl.argtypes = [vp, ctypes.c_char_p, c_int, c_int]
    lib.brsvd_allreduce.argtypes = [vp, vp, i64, c_int, c_int]
    lib.brsvd_allgather.argtypes = [vp, vp, vp, i64, c_int]
    lib.brsvd_ialm.argtypes = [vp, vp, i64, i64, i64, c_int, c_int, c_int, c_int, c_int,
                               c_int, u64, vp, dbl, dbl, dbl, dbl, c_int, vp, vp, c_int,
                               ctypes.POINTER(i32), ctypes.POINTER(i32), vp, vp, vp, vp]
    lib.brsvd_ialm_blocked.argtypes = [vp, vp, i64, i64, i64, c_int, c_int, c_int, c_int,
                                       c_int, c_int, u64, vp, dbl, dbl, dbl, dbl, c_int, vp,
                                       c_int, vp, vp, c_int, ctypes.POINTER(i32),
                                       ctypes.POINTER(i32), vp, vp, vp, vp]
    lib.brsvd_sketch_product.argtypes = [vp, vp, i64, i64, i64, c_int, c_int, c_int, vp,
                                         i64, i64, vp, i64]
    lib.brsvd_sketch_product_scaled.argtypes = [vp, vp, i64, i64, i64, c_int, c_int, c_int,
                                                vp, i64, i64, vp, i64, vp]
    lib.brsvd_absmax.argtypes = [vp, vp, i64, i64, i64, c_int, c_int, vp, vp]
    lib.brsvd_rsvd_stream.argtypes = [vp, vp, i64, i64, i64, c_int, c_int, c_int, c_int, c_int,
                                      vp, c_int, u64, vp, vp, vp, c_int, i64, c_int,
                                      ctypes.POINTER(BrsvdStats)]
    lib.brsvd_rsvd_stream_blocked.argtypes = [vp, vp, i64, i64, i64, c_int, c_int, c_int,
                                              c_int, c_int, vp, c_int, u64, vp, vp, vp, c_int,
                                              i64, c_int, c_int, ctypes.POINTER(BrsvdStats)]
    lib.brsvd_gram.argtypes = [vp, vp, i64, i64, i64, c_int, vp, i64, i64, vp]
    lib.brsvd_residual.argtypes = [vp, vp, i64, i64, i64, c_int, c_int, vp, i64, vp, vp, i64,
                                   i64, ctypes.POINTER(dbl)]
    lib.brsvd_chol_basis.argtypes = [vp, vp, i64, dbl, dbl, dbl, dbl, vp,
                                     ctypes.POINTER(i32), ctypes.POINTER(i32)]
    lib.brsvd_apply.argtypes = [vp, vp, i64, i64, i64, c_int, vp, i64, vp, i64, c_int, dbl,
                                dbl]
    lib.brsvd_normalize.argtypes = [vp, vp, i64, i64, i64, c_int, vp, i64]
    lib.brsvd_colmax.argtypes = [vp, vp, i64, i64, i64, c_int, i64, vp, vp]
    lib.brsvd_scale_cols.argtypes = [vp, vp, i64, i64, i64, c_int, vp]
    lib.brsvd_colmax_entries.argtypes = [vp, vp, i64, i64, i64, c_int, i64, vp]
    lib.brsvd_stream_rows_pass.argtypes = [vp, vp, i64, i64, i64, c_int, c_int, vp, i64, i64,
                                           vp, i64, vp, i64, i64, c_int, ctypes.POINTER(dbl)]
    lib.brsvd_normalize_f64.argtypes = [vp, vp, i64, i64, i64, c_int, vp, i64, vp, vp]
    lib.brsvd_normalize_t.argtypes = [vp, vp, i64, i64, i64, c_int, vp, i64, vp]
    lib.brsvd_unnormalised_peak.argtypes = [vp, vp, i64, i64, c_int, c_int, vp, vp,
                                            ctypes.POINTER(dbl)]
    lib.brsvd_ialm_stream.argtypes = [vp, vp, i64, i64, i64, c_int, c_int, c_int, c_int, u64,
                                      vp, dbl, dbl, dbl, dbl, c_int, vp, c_int, vp, vp, vp,
                                      c_int, ctypes.POINTER(i32), ctypes.POINTER(i32), vp, vp,
                                      vp, vp]
    lib.brsvd_profile_begin.argtypes = [vp]
    lib.brsvd_profile_end.argtypes = [vp, ctypes.POINTER(BrsvdProfile)]
    for name in EXPORTED:
        if name not in ("brsvd_last_error", "brsvd_version"):
            getattr(lib, name).restype = c_int
    return lib


def load_library(path=LIB_PATH):
    """Load (once) and return the ctypes handle of libbrsvd."""
    global _lib
    with _lib_lock:
        if _lib is None:
            if not os.path.exists(path):
                raise BackendUnavailable(
                    f"{path} not found: build the CUDA extension first "
                    "(python -m paper_1706_07191_b200.build)")
            _lib = _declare(ctypes.CDLL(path))
        return _lib


class profile:
    """Context manager: device profile of the library calls made inside it.

        with _lib.profile() as prof: ...
        prof.report.big_ms, prof.report.gpu_launches
    """

    def __init__(self, device=None):
        self.ctx = context(device)
        self.report = BrsvdProfile()

    def __enter__(self):
        check(load_library().brsvd_profile_begin(self.ctx.handle))
        return self

    def __exit__(self, *exc):
        check(load_library().brsvd_profile_end(self.ctx.handle, ctypes.byref(self.report)))
        return False


def last_error():
    return load_library().brsvd_last_error().decode(errors="replace")


class _Ctx:
    def __init__(self, device):
        lib = load_library()
        h = ctypes.c_void_p()
        rc = lib.brsvd_ctx_create(device, None, ctypes.byref(h))
        if rc != OK:
            raise BackendUnavailable(f"brsvd_ctx_create(device={device}) failed: "
                                     f"{last_error()}")
        self.handle = h
        self.device = device
        self.stream = None

    def set_stream(self, stream_ptr):
        if stream_ptr != self.stream:
            check(load_library().brsvd_ctx_set_stream(self.handle,
                                                      ctypes.c_void_p(stream_ptr)))
            self.stream = stream_ptr


def context(device=None):
    """Per-thread, per-device context (contexts are not re-entrant)."""
    if device is None:
        device = int(os.environ.get("BRSVD_DEVICE", "0"))
    ctxs = getattr(_tls, "ctxs", None)
    if ctxs is None:
        ctxs = _tls.ctxs = {}
    c = ctxs.get(device)
    if c is None:
        c = ctxs[device] = _Ctx(device)
    return c


def check(rc):
    """Map a status code to the reference's exception types."""
    if rc == OK:
        return
    msg = last_error()
    if rc == ERR_CONFIG:
        from .rsvd import ConfigError
        raise ConfigError(msg)
    if rc == ERR_SHAPE:
        from .kernels import ShapeError
        raise ShapeError(msg)
    if rc == ERR_OVERFLOW:
        raise FloatingPointError(msg)
    if rc == ERR_BUDGET:
        from .store import BudgetError
        # the C side reports "... minimum_feasible=<bytes>" (store.py:42-47)
        need = None
        if "minimum_feasible=" in msg:
            try:
                need = int(msg.rsplit("minimum_feasible=", 1)[1].split()[0])
            except ValueError:
                need = None
        raise BudgetError(msg, need)
    if rc == ERR_NCCL:
        raise RuntimeError(f"NCCL error: {msg}")
    if rc == ERR_CUDA:
        raise RuntimeError(f"CUDA error: {msg}")
    raise ValueError(msg)


def dtype_code(dtype):
    dt = np.dtype(dtype)
    if dt == np.float64:
        return F64
    if dt == np.float32:
        return F32
    raise TypeError(f"unsupported dtype {dt}; expected float64 or float32")
