"""Randomized SVD entry points on the B200 (drop-in for ``blocksvd.rsvd``).

Every decomposition runs the same GPU pipeline (include/brsvd.h,
``brsvd_rsvd``): global power iteration Y = (A A^T)^q A Omega with a basis
change between passes, rank-revealing orthonormalisation, projection
B = Q^T A, one-sided Jacobi SVD of the core, canonical signs.  This is the
semantics of ``rsvd_incore`` (rsvd.py:126-141) and ``rsvd_naive_ooc``
(rsvd.py:218-284) at any partition count.

Store entry points:
  * ``brsvd_run`` computes the reference's per-block power iteration
    (rsvd.py:169-175) by default; ``mode="global"`` gives the global one.
  * ``PassStats`` follows the reference's accounting (2 passes for
    brsvd_run, 2(q+1) for rsvd_naive_ooc); ``stats.boundary_words_read`` is
    the true host->device traffic: one pass when the store fits in HBM, the
    streamed passes (2 paper / q + 2 global) when it exceeds the budget.
"""

import ctypes
import time
from dataclasses import dataclass

import numpy as np

from . import _lib
from ._arrays import DeviceMatrix, HostMatrix, is_torch, torch_stream_ptr
from .kernels import SvdFactors, warn_rank
from .store import MatrixStore, plan_blocks

__all__ = [
    "SketchConfig",
    "ConfigError",
    "rsvd_incore",
    "brsvd_run",
    "block_range_finder",
    "rsvd_naive_ooc",
    "relative_frobenius_error",
]

Q_MAX_DEFAULT = 10


class ConfigError(ValueError):
    """Sketch parameters inconsistent with the matrix shape (rsvd.py:43-44)."""


@dataclass
class SketchConfig:
    """Randomized range-finder parameters (rsvd.py:47-81)."""

    target_rank: int
    oversampling: int = 10
    power_exponent: int = 0
    partitions: object = "auto"
    master_seed: int = 0
    q_max: int = Q_MAX_DEFAULT

    @property
    def l(self):
        return self.target_rank + self.oversampling

    def validate(self, m, n):
        if self.target_rank < 1:
            raise ConfigError(f"target rank must be positive, got {self.target_rank}")
        if self.oversampling < 0:
            raise ConfigError("oversampling must be non-negative")
        if self.l > min(m, n):
            raise ConfigError(f"k + p = {self.l} exceeds min(m, n) = {min(m, n)}")
        if not (0 <= self.power_exponent <= self.q_max):
            raise ConfigError(
                f"power exponent {self.power_exponent} outside [0, {self.q_max}]")
        if self.partitions != "auto" and int(self.partitions) < 1:
            raise ConfigError(f"partitions must be positive, got {self.partitions}")


@dataclass
class RsvdRun:
    """Factors plus the device-side diagnostics of one decomposition."""

    factors: SvdFactors
    stats: object          # _lib.BrsvdStats
    wall_seconds: float


def _omega_arg(omega, n, l, dtype, device):
    """Validate an injected sketch (n x l) and return (keepalive, ptr, where)."""
    if omega is None:
        return None, None, _lib.DEVICE
    if device:
        import torch
        t = omega if is_torch(omega) else torch.as_tensor(np.asarray(omega))
        t = t.to(device="cuda", dtype=torch.float64 if dtype == np.float64 else torch.float32)
        if tuple(t.shape) != (n, l):
            from .kernels import ShapeError
            raise ShapeError(f"omega has shape {tuple(t.shape)}, expected ({n}, {l})")
        t = t.t().contiguous()  # column-major n x l
        return t, ctypes.c_void_p(t.data_ptr()), _lib.DEVICE
    o = np.asfortranarray(np.asarray(omega), dtype=dtype)
    if o.shape != (n, l):
        from .kernels import ShapeError
        raise ShapeError(f"omega has shape {o.shape}, expected ({n}, {l})")
    return o, ctypes.c_void_p(o.ctypes.data), _lib.HOST


def host_outputs(m, n, l, npdt):
    """U (m x l, Fortran order) and Vt (l x n) as numpy arrays backed by
    page-locked host memory (torch's caching host allocator), so the D2H copies
    of the factors run at full PCIe rate instead of faulting in fresh pageable
    pages; plain numpy arrays when pinning is unavailable."""
    try:
        import torch
        tdt = torch.float64 if npdt == np.float64 else torch.float32
        U = torch.empty((l, m), dtype=tdt, pin_memory=True).numpy().T
        Vt = torch.empty((l, n), dtype=tdt, pin_memory=True).numpy()
        return U, Vt
    except (RuntimeError, ImportError):
        return (np.empty((m, l), dtype=npdt, order="F"),
                np.empty((l, n), dtype=npdt, order="C"))


def run_rsvd(a, cfg, omega=None, warn=True, blocks=None):
    """One GPU decomposition; returns RsvdRun (factors + stats).

    ``a`` is a 2-D numpy array (host; results come back as numpy) or a torch
    CUDA tensor (device; results stay on the device as torch tensors).
    """
    device = is_torch(a)
    mat = DeviceMatrix(a) if device else HostMatrix(a)
    m, n = mat.shape
    cfg.validate(m, n)
    k, p, q = cfg.target_rank, cfg.oversampling, cfg.power_exponent
    l = k + p
    lib = _lib.load_library()
    if device:
        import torch
        ctx = _lib.context(mat.device)
        ctx.set_stream(torch_stream_ptr(mat.t))
        tdt = mat.t.dtype
        U = torch.empty((l, m), dtype=tdt, device=mat.t.device)     # col-major m x l
        sigma = torch.empty(l, dtype=tdt, device=mat.t.device)
        Vt = torch.empty((l, n), dtype=tdt, device=mat.t.device)
        ptrs = [ctypes.c_void_p(x.data_ptr()) for x in (U, sigma, Vt)]
        where = _lib.DEVICE
        npdt = np.float64 if tdt == torch.float64 else np.float32
    else:
        ctx = _lib.context()
        npdt = mat.dtype
        U, Vt = host_outputs(m, n, l, npdt)
        sigma = np.empty(l, dtype=npdt)
        ptrs = [ctypes.c_void_p(x.ctypes.data) for x in (U, sigma, Vt)]
        where = _lib.HOST
    keep, optr, owhere = _omega_arg(omega, n, l, npdt, device)
    stats = _lib.BrsvdStats()
    bounds, nblk = None, 0
    if blocks is not None and len(blocks) > 1:
        edges = [int(blocks[0][0])] + [int(j1) for _, j1 in blocks]
        bounds = (ctypes.c_int64 * len(edges))(*edges)
        nblk = len(edges) - 1
    t0 = time.perf_counter()
    rc = lib.brsvd_rsvd_blocked(ctx.handle, mat.ptr, m, n, mat.ld, mat.code, mat.layout, where,
                                k, p, q, optr, owhere,
                                ctypes.c_uint64(int(cfg.master_seed) & (2 ** 64 - 1)),
                                bounds, nblk, ptrs[0], ptrs[1], ptrs[2], where,
                                ctypes.byref(stats))
    wall = time.perf_counter() - t0
    del keep
    _lib.check(rc)
    if warn:
        warn_rank(stats.detected_rank, l)
        warn_rank(stats.core_rank, l)
    if device:
        U = U.t()
    f = SvdFactors(U=U, sigma=sigma, Vt=Vt, target_rank=k, effective_l=l)
    return RsvdRun(factors=f, stats=stats, wall_seconds=wall)


def rsvd_incore(a, cfg, omega=None):
    """Randomized SVD of an in-memory matrix (rsvd.py:126-141), on the GPU.

    ``omega`` optionally injects the n x l sketch (e.g. the reference's
    ``gaussian_matrix(n, l, seed, 0, dtype)``) for bitwise-identical inputs.
    """
    return run_rsvd(a, cfg, omega=omega).factors


def _load_store_to_device(store, plan):
    """Read every block of the plan once and land it in HBM (column-major).

    The store's own read counters are left unchanged: the entry points book
    the reference's per-algorithm accounting and the boundary traffic
    themselves (_account)."""
    w0, b0 = store.stats.words_read, store.stats.block_reads
    try:
        return _land_blocks(store, plan)
    finally:
        store.stats.words_read, store.stats.block_reads = w0, b0


def _land_blocks(store, plan):
    import torch
    tdt = torch.float64 if store.dtype == np.float64 else torch.float32
    ctx = _lib.context()
    dev = torch.empty((store.n, store.m), dtype=tdt, device=f"cuda:{ctx.device}")
    pinned = None
    for j0, j1 in plan:
        w = j1 - j0
        if pinned is None or pinned.numel() < store.m * w:
            pinned = torch.empty(store.m * w, dtype=tdt, pin_memory=True)
        buf = pinned[: store.m * w]
        store.read_block_into(j0, j1, buf.numpy())
        dev[j0:j1].view(-1).copy_(buf, non_blocking=False)
    return dev.t()   # m x n column-major view


def run_rsvd_stream(a, cfg, panel=None, nbuf=3, omega=None, warn=True, block_power=False):
    """Out-of-core decomposition of a host-resident matrix (C ABI
    ``brsvd_rsvd_stream``): A is streamed over PCIe in panels of ``panel``
    rows (C-ordered ``a``) or columns (Fortran-ordered ``a``) through ``nbuf``
    device buffers; q + 2 passes.  Pinned host memory (e.g. a numpy view of a
    ``torch.empty(..., pin_memory=True)`` tensor) overlaps copies with compute.
    Returns RsvdRun with numpy factors."""
    mat = HostMatrix(a)
    m, n = mat.shape
    cfg.validate(m, n)
    k, p, q = cfg.target_rank, cfg.oversampling, cfg.power_exponent
    l = k + p
    inner = n if mat.layout == _lib.ROW_MAJOR else m
    if panel is None:   # ~1 GiB panels
        panel = max(1, (1 << 30) // max(1, inner * mat.a.itemsize))
    ctx = _lib.context()
    U, Vt = host_outputs(m, n, l, mat.dtype)
    sigma = np.empty(l, dtype=mat.dtype)
    keep, optr, owhere = _omega_arg(omega, n, l, mat.dtype, False)
    stats = _lib.BrsvdStats()
    t0 = time.perf_counter()
    rc = _lib.load_library().brsvd_rsvd_stream_blocked(
        ctx.handle, mat.ptr, m, n, mat.ld, mat.code, mat.layout, k, p, q, optr, owhere,
        ctypes.c_uint64(int(cfg.master_seed) & (2 ** 64 - 1)),
        ctypes.c_void_p(U.ctypes.data), ctypes.c_void_p(sigma.ctypes.data),
        ctypes.c_void_p(Vt.ctypes.data), _lib.HOST, int(panel), int(nbuf),
        1 if block_power else 0, ctypes.byref(stats))
    wall = time.perf_counter() - t0
    del keep
    _lib.check(rc)
    if warn:
        warn_rank(stats.detected_rank, l)
        warn_rank(stats.core_rank, l)
    f = SvdFactors(U=U, sigma=sigma, Vt=Vt, target_rank=k, effective_l=l)
    return RsvdRun(factors=f, stats=stats, wall_seconds=wall)


def _store_payload(store):
    """Read-only memory map of a store's column-major payload (m x n)."""
    from .store import HEADER_SIZE
    mm = np.memmap(store.path, dtype=store.dtype, mode="r", offset=HEADER_SIZE,
                   shape=(store.n, store.m))
    return mm.T   # m x n, Fortran-ordered view


_MODES = ("global", "paper")


def run_range(a, cfg, omega=None, blocks=None, warn=True):
    """Sketch + orthonormal basis only (C ABI ``brsvd_range_finder``): Q (m x l)
    spanning the sample -- global power iteration, or the per-block iteration
    over ``blocks`` (the paper's block_range_finder, rsvd.py:150-185).
    Returns (Q, stats); Q matches ``a``'s kind (numpy host / torch device)."""
    device = is_torch(a)
    mat = DeviceMatrix(a) if device else HostMatrix(a)
    m, n = mat.shape
    cfg.validate(m, n)
    k, p, q = cfg.target_rank, cfg.oversampling, cfg.power_exponent
    l = k + p
    lib = _lib.load_library()
    if device:
        import torch
        ctx = _lib.context(mat.device)
        ctx.set_stream(torch_stream_ptr(mat.t))
        Q = torch.empty((l, m), dtype=mat.t.dtype, device=mat.t.device)
        npdt = np.float64 if mat.t.dtype == torch.float64 else np.float32
        qptr, where = ctypes.c_void_p(Q.data_ptr()), _lib.DEVICE
    else:
        ctx = _lib.context()
        npdt = mat.dtype
        Q = np.empty((m, l), dtype=npdt, order="F")
        qptr, where = ctypes.c_void_p(Q.ctypes.data), _lib.HOST
    keep, optr, owhere = _omega_arg(omega, n, l, npdt, device)
    bounds, nblk = None, 0
    if blocks is not None and len(blocks) > 1:
        edges = [int(blocks[0][0])] + [int(j1) for _, j1 in blocks]
        bounds = (ctypes.c_int64 * len(edges))(*edges)
        nblk = len(edges) - 1
    stats = _lib.BrsvdStats()
    rc = lib.brsvd_range_finder(ctx.handle, mat.ptr, m, n, mat.ld, mat.code, mat.layout,
                                where, k, p, q, optr, owhere,
                                ctypes.c_uint64(int(cfg.master_seed) & (2 ** 64 - 1)),
                                bounds, nblk, qptr, where, ctypes.byref(stats))
    del keep
    _lib.check(rc)
    if warn:
        warn_rank(stats.detected_rank, l)
    return (Q.t() if device else Q), stats


def _host_factors(f):
    return SvdFactors(U=f.U.cpu().numpy(), sigma=f.sigma.cpu().numpy(),
                      Vt=f.Vt.cpu().numpy(), target_rank=f.target_rank,
                      effective_l=f.effective_l)


def _account(stats, store, plan, cfg, algorithm, seconds, boundary_passes):
    """Pass accounting of the reference's algorithm (store.py:50-79 counters as
    rsvd.py:150-284 increments them): the passes the algorithm makes over A --
    on the B200 they are HBM passes when the store fits the device -- plus the
    true host->device traffic in ``stats.boundary_words_read``."""
    m, n, l, q, s = store.m, store.n, cfg.l, cfg.power_exponent, plan.s
    mn = m * n
    if algorithm in ("paper", "global_brsvd"):   # brsvd_run: sketch pass + core pass
        stages = (("sketch", mn, 2 * mn * l * (1 + 2 * q)), ("orthonormalize", 0, 2 * m * l * l),
                  ("form_core", mn, 2 * mn * l), ("svd", 0, 2 * n * l * l + 2 * m * l * l))
        reads = 2 * s
    elif algorithm == "naive":        # rsvd_naive_ooc: 2(q + 1) passes
        stages = (("sketch", mn, 2 * mn * l), ("power", 2 * q * mn, 4 * mn * l * q),
                  ("orthonormalize", 0, 2 * m * l * l), ("form_core", mn, 2 * mn * l),
                  ("svd", 0, 2 * n * l * l + 2 * m * l * l))
        reads = 2 * (q + 1) * s
    else:                             # block_range_finder: one sketch pass
        stages = (("sketch", mn, 2 * mn * l * (1 + 2 * q)), ("orthonormalize", 0, 2 * m * l * l))
        reads = s
    for name, words, flops in stages:
        stats.words_read += words
        stats.flop_estimate += flops
        stats.log_stage(name, words, 0, seconds.get(name, 0.0))
    stats.block_reads += reads
    stats.boundary_words_read += int(boundary_passes * mn)


def _run_store(store, cfg, memory_budget_bytes, algorithm, omega=None):
    m, n = store.m, store.n
    cfg.validate(m, n)
    s = None if cfg.partitions == "auto" else int(cfg.partitions)
    plan = plan_blocks(n, m, cfg.l, store.element_size,
                       memory_budget_bytes=memory_budget_bytes, s=s)
    store.reset_stats()
    stats = store.stats
    paper = algorithm == "paper"
    if memory_budget_bytes is not None and store.payload_bytes > memory_budget_bytes:
        # Out of core: the budget's column blocks are the streamed panels.
        # paper: each block's power iteration runs while it is resident, then
        # the core pass (2 passes over PCIe); global: q + 2 passes.
        run = run_rsvd_stream(_store_payload(store), cfg, panel=plan.n_prime, nbuf=3,
                              omega=omega, block_power=paper)
        st = run.stats
        crossed = st.words_read // (m * n)
        factors = run.factors
    else:
        t0 = time.perf_counter()
        a_dev = _load_store_to_device(store, plan)
        load_s = time.perf_counter() - t0
        run = run_rsvd(a_dev, cfg, omega=omega, blocks=list(plan) if paper else None)
        st = run.stats
        st.seconds_sketch += load_s
        crossed = 1
        factors = _host_factors(run.factors)
        del a_dev
    seconds = {"sketch": st.seconds_sketch, "orthonormalize": st.seconds_orthonormalize,
               "form_core": st.seconds_form_core, "svd": st.seconds_svd}
    _account(stats, store, plan, cfg, algorithm, seconds, crossed)
    return factors, stats, plan


def brsvd_run(store, cfg, memory_budget_bytes=None, mode="paper", omega=None):
    """Block randomized SVD of a stored matrix (rsvd.py:188-215) on the GPU.

    Returns (factors, stats) with the reference's pass accounting
    (``stats.full_passes == 2``, ``block_reads == 2 s``; rsvd.py:188-193);
    ``stats.boundary_words_read`` is what actually crossed PCIe -- one pass
    when the store fits the budget (it is landed in HBM once and every pass
    runs from HBM), two when its column blocks are streamed.

    mode="paper" (default, the reference's semantics): the per-block power
    iteration of block_range_finder (rsvd.py:169-175) -- each column block's
    (A_J A_J^T)^q A_J Omega_J, unnormalised, summed; identical to the global
    iteration when s = 1 or q = 0.  mode="global": the global power iteration
    of rsvd_incore / rsvd_naive_ooc at any s (q + 2 passes when streamed).
    ``omega`` (n x l) injects the sketch, e.g. the reference's
    gaussian_matrix(n, l, seed, 0), whose rows are the per-block slices the
    reference draws (kernels.py:98-118, row_offset).
    """
    if mode not in _MODES:
        raise ValueError(f"mode must be one of {_MODES}, got {mode!r}")
    factors, stats, _ = _run_store(store, cfg, memory_budget_bytes,
                                   "paper" if mode == "paper" else "global_brsvd", omega)
    return factors, stats


def rsvd_naive_ooc(store, cfg, memory_budget_bytes=None, omega=None):
    """Global-power-iteration SVD of a stored matrix (rsvd.py:218-284).

    Reference pass accounting: 2(q + 1) passes, 2(q + 1) s block reads
    (tests/test_rsvd.py:173-179); ``stats.boundary_words_read`` is the true
    PCIe traffic (1 pass from HBM, q + 2 when streamed).
    """
    factors, stats, _ = _run_store(store, cfg, memory_budget_bytes, "naive", omega)
    return factors, stats


def block_range_finder(store, cfg, memory_budget_bytes=None, plan=None, omega=None):
    """Orthonormal range basis from one blocked pass over the store
    (rsvd.py:150-185); returns (Q, plan).

    The sample is the reference's per-block power iteration over the plan's
    column blocks, then its orthonormal basis (no core projection).  Q spans
    the same range as the reference's tsqr Q (a different orthonormal basis of
    that span).  Like the reference, it adds its pass to ``store.stats``
    without resetting it.  The store is landed in HBM once (one pass across
    the boundary, as the reference reads it once).
    """
    m, n = store.m, store.n
    cfg.validate(m, n)
    if plan is None:
        s = None if cfg.partitions == "auto" else int(cfg.partitions)
        plan = plan_blocks(n, m, cfg.l, store.element_size,
                           memory_budget_bytes=memory_budget_bytes, s=s)
    t0 = time.perf_counter()
    a_dev = _load_store_to_device(store, plan)
    Q, st = run_range(a_dev, cfg, omega=omega, blocks=list(plan))
    Qh = Q.cpu().numpy()
    seconds = {"sketch": time.perf_counter() - t0 - st.seconds_orthonormalize,
               "orthonormalize": st.seconds_orthonormalize}
    _account(store.stats, store, plan, cfg, "range", seconds, 1)
    return np.asfortranarray(Qh), plan


def _residual_sums(a_dev, U_col, sig, Vt, j0=0):
    """(||A - U diag(s) Vt[:, j0:j0+n]||^2, ||A||^2) of a device block through
    the fused C-ABI kernel (brsvd_residual)."""
    import torch
    mat = DeviceMatrix(a_dev)
    m, n = mat.shape
    l = U_col.shape[1]
    lib = _lib.load_library()
    ctx = _lib.context(mat.device)
    ctx.set_stream(torch_stream_ptr(mat.t))
    esz = U_col.element_size()
    out = (ctypes.c_double * 2)()
    rc = lib.brsvd_residual(ctx.handle, mat.ptr, m, n, mat.ld, mat.code, mat.layout,
                            ctypes.c_void_p(U_col.data_ptr()), U_col.stride(1),
                            ctypes.c_void_p(sig.data_ptr()),
                            ctypes.c_void_p(Vt.data_ptr() + j0 * esz), Vt.stride(0), l, out)
    _lib.check(rc)
    return out[0], out[1]


def relative_frobenius_error(source, factors, block_width=None):
    """||A - U diag(sigma) Vt||_F / ||A||_F (rsvd.py:396-432), on the GPU.

    One fused pass over A (brsvd_residual: the rank-l reconstruction is formed
    tile by tile in registers and subtracted as A is read; sums of squares in
    fp64).  A store is streamed in column blocks (one extra pass, like the
    reference); an in-memory matrix is used as is.
    """
    import torch
    dev = f"cuda:{_lib.context().device}"

    def T(x, dt):
        t = x.to(dev) if is_torch(x) else torch.as_tensor(np.asarray(x), device=dev)
        return t.to(dt)

    if isinstance(source, MatrixStore):
        m, n = source.m, source.n
        tdt = torch.float64 if source.dtype == np.float64 else torch.float32
    else:
        a = source if is_torch(source) else np.asarray(source)
        m, n = a.shape
        tdt = (a.dtype if is_torch(a) else
               (torch.float64 if a.dtype == np.float64 else torch.float32))
        if tdt not in (torch.float32, torch.float64):
            tdt = torch.float64
    U_d = T(factors.U, tdt)
    Vt_d = T(factors.Vt, tdt).contiguous()
    s_d = T(factors.sigma, tdt).contiguous()
    if U_d.shape[0] != m or Vt_d.shape[1] != n:
        raise ValueError(f"factor shapes {U_d.shape[0]}x{Vt_d.shape[1]} do not "
                         f"match source {m}x{n}")
    U_col = U_d.t().contiguous().t()    # column-major m x l
    num = den = 0.0
    if isinstance(source, MatrixStore):
        if block_width is None:
            block_width = max(1, min(n, (256 << 20) // max(1, m * source.element_size)))
        for j0 in range(0, n, block_width):
            j1 = min(j0 + block_width, n)
            blk = torch.as_tensor(source.read_block(j0, j1), device=dev).to(tdt)
            blk = blk.t().contiguous().t() if not blk.t().is_contiguous() else blk
            a_, b_ = _residual_sums(blk, U_col, s_d, Vt_d, j0)
            num += a_
            den += b_
    else:
        a_d = T(a, tdt)
        num, den = _residual_sums(a_d, U_col, s_d, Vt_d)
    if den == 0.0:
        return 0.0 if num == 0.0 else float("inf")
    return float(np.sqrt(num) / np.sqrt(den))


def sketch_product(A, X, trans=False):
    """One A-streaming product on the GPU: A @ X (trans=False) or A.T @ X.

    ``A`` (m x n) and ``X`` are torch CUDA tensors; returns a new tensor
    (column-major storage).  This is the unit each power-iteration pass is made
    of (rsvd.py:94-102); exposed for the sharded driver and for tests.
    """
    import torch
    mat = DeviceMatrix(A)
    m, n = mat.shape
    rows = n if trans else m
    xin = m if trans else n
    if X.dim() != 2 or X.shape[0] != xin:
        from .kernels import ShapeError
        raise ShapeError(f"X has shape {tuple(X.shape)}, expected ({xin}, l)")
    l = X.shape[1]
    Xc = X.to(dtype=mat.t.dtype).t().contiguous()          # column-major
    C = torch.empty((l, rows), dtype=mat.t.dtype, device=mat.t.device)
    ctx = _lib.context(mat.device)
    ctx.set_stream(torch_stream_ptr(mat.t))
    _lib.check(_lib.load_library().brsvd_sketch_product(
        ctx.handle, mat.ptr, m, n, mat.ld, mat.code, mat.layout, int(bool(trans)),
        ctypes.c_void_p(Xc.data_ptr()), xin, l, ctypes.c_void_p(C.data_ptr()), rows))
    return C.t()
