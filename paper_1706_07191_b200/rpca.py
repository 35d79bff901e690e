"""Robust PCA by inexact ALM with a randomized inner SVD, on the B200.

Drop-in for ``blocksvd.rpca`` (rpca.py): same configuration/result types and
solver semantics (rpca.py:168-213).  The whole iteration -- spectral-norm
estimate, randomized SVD of the iterate, singular-value shrinkage, the fused
low-rank/sparse/dual update and the residual -- runs on the GPU behind
``brsvd_ialm`` (include/brsvd.h); the host only checks the stopping rule the
library reports.
"""

import ctypes
import json
import os
import tempfile
from dataclasses import dataclass, field

import numpy as np

from . import _lib
from ._arrays import DeviceMatrix, HostMatrix, is_torch, torch_stream_ptr
from .store import BudgetError, MatrixStore, plan_blocks

__all__ = ["RpcaConfig", "RpcaResult", "shrink", "spectral_norm_estimate",
           "ialm_rpca"]


def shrink(x, epsilon):
    """Soft-thresholding sign(x) * max(|x| - eps, 0) (rpca.py:35-45).

    Works on scalars, numpy arrays and torch tensors; shape is preserved.
    """
    if epsilon < 0:
        raise ValueError(f"shrinkage threshold must be non-negative, got {epsilon}")
    if is_torch(x):
        import torch
        return torch.sign(x) * torch.clamp(torch.abs(x) - epsilon, min=0.0)
    x = np.asarray(x)
    out = np.sign(x) * np.maximum(np.abs(x) - epsilon, 0.0)
    return out if out.ndim else float(out)


@dataclass
class RpcaConfig:
    """Solver parameters (rpca.py:103-133)."""

    target_rank: int
    oversampling: int = 10
    power_exponent: int = 1
    lam: float = None
    mu0: float = None
    rho: float = 1.5
    tol: float = 1e-7
    max_iterations: int = 100
    master_seed: int = 0
    memory_budget_bytes: int = None

    def validate(self):
        if self.lam is not None and self.lam <= 0:
            raise ValueError("lambda must be positive")
        if self.mu0 is not None and self.mu0 <= 0:
            raise ValueError("mu0 must be positive")
        if self.rho <= 1:
            raise ValueError("rho must exceed 1")
        if self.tol <= 0:
            raise ValueError("tol must be positive")
        if self.max_iterations < 1:
            raise ValueError("max_iterations must be positive")


@dataclass
class RpcaResult:
    """Low-rank / sparse split with the convergence trace (rpca.py:136-150)."""

    L: object
    S: object
    iterations: int
    residual_history: list
    converged: bool
    history: list = field(default_factory=list)

    def to_json_lines(self):
        return "\n".join(json.dumps(e) for e in self.history)


def _require(name):
    lib = _lib.load_library()
    if not hasattr(lib, name):
        raise _lib.BackendUnavailable(f"{name} missing from {_lib.LIB_PATH}")
    return getattr(lib, name)


def spectral_norm_estimate(source, seed=0, tol=1e-10, max_iterations=100, start=None):
    """Largest singular value by power iteration on M^T M (rpca.py:72-100).

    Runs on the GPU; a zero matrix returns 0 with a warning.  ``start``
    (n values) injects the start vector -- the reference's
    ``gaussian_matrix(n, 1, seed, stream_index=7)[:, 0]`` for parity -- in place
    of this library's stream-7 sketch column (it is normalised here, as the
    reference does).
    """
    import warnings
    if isinstance(source, MatrixStore):
        source = source.read_full()
    mat = DeviceMatrix(source) if is_torch(source) else HostMatrix(source, "M")
    m, n = mat.shape
    fn = _require("brsvd_spectral_norm_start")
    ctx = _lib.context(getattr(mat, "device", None))
    st = None
    if start is not None:
        st = np.ascontiguousarray(np.asarray(start, dtype=np.float64).reshape(-1))
        if st.shape[0] != n:
            from .kernels import ShapeError
            raise ShapeError(f"start has {st.shape[0]} entries, expected {n}")
    if is_torch(source):
        ctx.set_stream(torch_stream_ptr(mat.t))
    out = ctypes.c_double()
    iters = ctypes.c_int32()
    _lib.check(fn(ctx.handle, mat.ptr, m, n, mat.ld, mat.code, mat.layout,
                  _lib.DEVICE if is_torch(source) else _lib.HOST,
                  ctypes.c_uint64(int(seed) & (2 ** 64 - 1)),
                  None if st is None else ctypes.c_void_p(st.ctypes.data), ctypes.c_double(tol),
                  int(max_iterations), ctypes.byref(out), ctypes.byref(iters)))
    if out.value == 0.0:
        warnings.warn("spectral_norm_estimate: zero matrix")
        return 0.0
    return float(out.value)


# device residency of the IALM loop: M, S, Y, W and the L/S outputs, plus slack
_IALM_RESIDENT_COPIES = 6


def _require_device_room(payload_bytes):
    """In-memory inputs keep the IALM iterates in HBM: one whose iterates
    cannot be held on the device raises BudgetError up front (store.py:42-47
    semantics) instead of failing inside the loop (stores take the streamed
    path instead, _ialm_stream)."""
    import torch
    free, _ = torch.cuda.mem_get_info(_lib.context().device)
    need = _IALM_RESIDENT_COPIES * int(payload_bytes)
    if need > free:
        raise BudgetError(
            f"IALM iterates of a {payload_bytes} B matrix need ~{need} B of device memory, "
            f"{free} B free (pass a MatrixStore with a memory budget to stream it)", need)


def _pinned_cm(m, n, dtype):
    """Column-major (m x n) host array in page-locked memory when possible."""
    try:
        import torch
        tdt = torch.float64 if np.dtype(dtype) == np.float64 else torch.float32
        return torch.empty((n, m), dtype=tdt, pin_memory=True).numpy().T
    except (RuntimeError, ImportError):
        return np.empty((m, n), dtype=dtype, order="F")


def _host_room(nbytes):
    """True when nbytes fit comfortably in the host's available memory."""
    try:
        import psutil
        return nbytes <= 0.7 * psutil.virtual_memory().available
    except ImportError:
        return False


def _ialm_stream(store, cfg, blocks, omega=None, nslots=2, pinned=None):
    """The reference's out-of-core branch (_ialm_rpca_ooc, rpca.py:216-304)
    with M, S and Y streamed block by block every pass (brsvd_ialm_stream);
    returns L and S as stores like the reference.

    pinned=None: when M, S, Y, L fit in host memory they live in page-locked
    buffers (overlapped DMA); otherwise -- a store beyond host RAM, the case
    the reference's branch exists for -- M is streamed straight from the
    store's memory map and S, Y, L are file-backed maps in a temporary
    directory, like the reference's temporary stores (rpca.py:240-243)."""
    from .rsvd import _store_payload
    from .store import HEADER_SIZE
    m, n = store.m, store.n
    dt = store.dtype
    payload = _store_payload(store)          # read-only memory map, m x n, Fortran order
    if pinned is None:
        pinned = _host_room(4 * store.payload_bytes)
    workdir = tempfile.mkdtemp(prefix="rpca_")
    w0, b0 = store.stats.words_read, store.stats.block_reads
    if pinned:
        M = _pinned_cm(m, n, dt)
        for j0, j1 in blocks:                # one read of the store into pinned memory
            M[:, j0:j1] = payload[:, j0:j1]
        S, Y, L = (_pinned_cm(m, n, dt) for _ in range(3))
        Ls = Ss = None
    else:
        M = payload
        Ls = MatrixStore.create(os.path.join(workdir, "lowrank.oocm"), m, n, dt)
        Ss = MatrixStore.create(os.path.join(workdir, "sparse.oocm"), m, n, dt)
        Ls.close()
        Ss.close()

        maps = [np.memmap(os.path.join(workdir, "lowrank.oocm"), dtype=dt, mode="r+",
                          offset=HEADER_SIZE, shape=(n, m)),
                np.memmap(os.path.join(workdir, "sparse.oocm"), dtype=dt, mode="r+",
                          offset=HEADER_SIZE, shape=(n, m)),
                np.memmap(os.path.join(workdir, "dual.bin"), dtype=dt, mode="w+",
                          shape=(n, m))]
        L, S, Y = (mm.T for mm in maps)       # m x n, Fortran order
    store.stats.words_read, store.stats.block_reads = w0 + m * n, b0 + len(blocks)
    maxit = int(cfg.max_iterations)
    res, mus, svd_s, it_s = (np.zeros(maxit) for _ in range(4))
    iters, conv = ctypes.c_int32(), ctypes.c_int32()
    l = int(cfg.target_rank) + int(cfg.oversampling)
    om, optr = None, None
    if omega is not None:
        if tuple(np.shape(omega)) != (n, l):
            raise ValueError(f"omega has shape {np.shape(omega)}, expected ({n}, {l})")
        om = np.asfortranarray(np.asarray(omega), dtype=dt)
        optr = ctypes.c_void_p(om.ctypes.data)
    edges = [int(blocks[0][0])] + [int(j1) for _, j1 in blocks]
    bounds = (ctypes.c_int64 * len(edges))(*edges)
    nan = float("nan")
    dptr = lambda a: ctypes.c_void_p(a.ctypes.data)  # noqa: E731
    _lib.check(_require("brsvd_ialm_stream")(
        _lib.context().handle, dptr(M), m, n, m, _lib.dtype_code(dt),
        int(cfg.target_rank), int(cfg.oversampling), int(cfg.power_exponent),
        ctypes.c_uint64(int(cfg.master_seed) & (2 ** 64 - 1)), optr,
        ctypes.c_double(nan if cfg.lam is None else float(cfg.lam)),
        ctypes.c_double(nan if cfg.mu0 is None else float(cfg.mu0)),
        ctypes.c_double(float(cfg.rho)), ctypes.c_double(float(cfg.tol)), maxit,
        bounds, len(edges) - 1, dptr(L), dptr(S), dptr(Y), int(nslots),
        ctypes.byref(iters), ctypes.byref(conv), dptr(res), dptr(mus), dptr(svd_s),
        dptr(it_s)))
    k = iters.value
    history = [{"i": i + 1, "mu": float(mus[i]), "residual": float(res[i]),
                "svd_seconds": float(svd_s[i]), "iter_seconds": float(it_s[i])}
               for i in range(k)]
    if pinned:
        Ls = MatrixStore.from_array(os.path.join(workdir, "lowrank.oocm"), L)
        Ss = MatrixStore.from_array(os.path.join(workdir, "sparse.oocm"), S)
    else:
        for mm in maps:
            mm.flush()
        del L, S, Y, maps
        os.remove(os.path.join(workdir, "dual.bin"))
        Ls = MatrixStore(os.path.join(workdir, "lowrank.oocm"))
        Ss = MatrixStore(os.path.join(workdir, "sparse.oocm"))
    return RpcaResult(L=Ls, S=Ss, iterations=k, residual_history=[float(r) for r in res[:k]],
                      converged=bool(conv.value), history=history)


def _device_room(payload_bytes):
    import torch
    free, _ = torch.cuda.mem_get_info(_lib.context().device)
    return _IALM_RESIDENT_COPIES * int(payload_bytes) <= free


def ialm_rpca(m_input, cfg, omega=None, stream=None, pinned=None):
    """Inexact-ALM robust PCA with a randomized inner SVD (rpca.py:153-213).

    Non-convergence at max_iterations returns ``converged=False``.  numpy (or
    store) input gives numpy output; a torch CUDA tensor keeps everything on
    the device.  When the reference would take its out-of-core branch
    (store payload above ``memory_budget_bytes``, rpca.py:160-163) the split
    is returned as MatrixStore objects as it does.  ``omega`` optionally
    injects the n x (k+p) sketch used by every inner SVD (parity runs pass the
    reference's ``gaussian_matrix(n, k+p, seed, 0, dtype)``).  ``stream``
    (out-of-core branch only): True streams M, S, Y from host memory block by
    block every pass (brsvd_ialm_stream); None does so when the iterates do not
    fit in device memory, else they are held in HBM.
    """
    cfg.validate()
    as_stores = False
    blocks = None
    if isinstance(m_input, MatrixStore):
        budget = cfg.memory_budget_bytes
        as_stores = budget is not None and m_input.payload_bytes > budget
        if as_stores:
            # the reference's out-of-core branch calls brsvd_run(W, sketch,
            # memory_budget_bytes=budget) (rpca.py:274): the inner SVDs use the
            # per-block power iteration over that plan's column blocks
            l_ = int(cfg.target_rank) + int(cfg.oversampling)
            plan = plan_blocks(m_input.n, m_input.m, l_, m_input.element_size,
                               memory_budget_bytes=budget)
            blocks = list(plan)
            # iterates that fit in HBM stay there (one read of the store);
            # beyond that (or stream=True) M, S, Y are streamed per pass
            if stream is None:
                stream = not _device_room(m_input.payload_bytes)
            if stream:
                return _ialm_stream(m_input, cfg, blocks, omega, pinned=pinned)
        _require_device_room(m_input.payload_bytes)
        m_input = m_input.read_full()
    device = is_torch(m_input)
    mat = DeviceMatrix(m_input) if device else HostMatrix(m_input, "M")
    m, n = mat.shape
    fn = _require("brsvd_ialm_blocked")
    ctx = _lib.context(getattr(mat, "device", None))
    maxit = int(cfg.max_iterations)
    if device:
        import torch
        ctx.set_stream(torch_stream_ptr(mat.t))
        # outputs share the input layout
        if mat.layout == _lib.ROW_MAJOR:
            L = torch.empty((m, n), dtype=mat.t.dtype, device=mat.t.device)
            S = torch.empty((m, n), dtype=mat.t.dtype, device=mat.t.device)
        else:
            L = torch.empty((n, m), dtype=mat.t.dtype, device=mat.t.device).t()
            S = torch.empty((n, m), dtype=mat.t.dtype, device=mat.t.device).t()
        lp, sp = ctypes.c_void_p(L.data_ptr()), ctypes.c_void_p(S.data_ptr())
        where = _lib.DEVICE
    else:
        order = "C" if mat.layout == _lib.ROW_MAJOR else "F"
        L = np.empty((m, n), dtype=mat.dtype, order=order)
        S = np.empty((m, n), dtype=mat.dtype, order=order)
        lp, sp = ctypes.c_void_p(L.ctypes.data), ctypes.c_void_p(S.ctypes.data)
        where = _lib.HOST
    res = np.zeros(maxit, dtype=np.float64)
    mus = np.zeros(maxit, dtype=np.float64)
    svd_s = np.zeros(maxit, dtype=np.float64)
    it_s = np.zeros(maxit, dtype=np.float64)
    iters = ctypes.c_int32()
    conv = ctypes.c_int32()
    nan = float("nan")
    l = int(cfg.target_rank) + int(cfg.oversampling)
    if omega is not None:
        if device:
            import torch
            om = torch.as_tensor(np.asarray(omega) if not is_torch(omega) else omega)
            om = om.to(device=mat.t.device, dtype=mat.t.dtype).t().contiguous()
            optr = ctypes.c_void_p(om.data_ptr())
        else:
            om = np.asfortranarray(np.asarray(omega), dtype=mat.dtype)
            optr = ctypes.c_void_p(om.ctypes.data)
        if tuple(np.shape(omega)) != (n, l):
            raise ValueError(f"omega has shape {np.shape(omega)}, expected ({n}, {l})")
    else:
        om, optr = None, None
    dptr = lambda a: ctypes.c_void_p(a.ctypes.data)  # noqa: E731
    bounds, nblk = None, 0
    if blocks is not None and len(blocks) > 1:
        edges = [int(blocks[0][0])] + [int(j1) for _, j1 in blocks]
        bounds = (ctypes.c_int64 * len(edges))(*edges)
        nblk = len(edges) - 1
    _lib.check(fn(
        ctx.handle, mat.ptr, m, n, mat.ld, mat.code, mat.layout, where,
        int(cfg.target_rank), int(cfg.oversampling), int(cfg.power_exponent),
        ctypes.c_uint64(int(cfg.master_seed) & (2 ** 64 - 1)), optr,
        ctypes.c_double(nan if cfg.lam is None else float(cfg.lam)),
        ctypes.c_double(nan if cfg.mu0 is None else float(cfg.mu0)),
        ctypes.c_double(float(cfg.rho)), ctypes.c_double(float(cfg.tol)), maxit,
        bounds, nblk, lp, sp, where, ctypes.byref(iters), ctypes.byref(conv),
        dptr(res), dptr(mus), dptr(svd_s), dptr(it_s)))
    k = iters.value
    residuals = [float(r) for r in res[:k]]
    history = [{"i": i + 1, "mu": float(mus[i]), "residual": float(res[i]),
                "svd_seconds": float(svd_s[i]), "iter_seconds": float(it_s[i])}
               for i in range(k)]
    if as_stores:
        workdir = tempfile.mkdtemp(prefix="rpca_")
        L = MatrixStore.from_array(os.path.join(workdir, "lowrank.oocm"), L)
        S = MatrixStore.from_array(os.path.join(workdir, "sparse.oocm"), S)
    return RpcaResult(L=L, S=S, iterations=k, residual_history=residuals,
                      converged=bool(conv.value), history=history)
