"""Row-sharded randomized SVD over several GPUs (BASELINE config 4).

The rows of A are split in contiguous panels, one per rank:
rank g holds A[r0:r1, :], its rows of the sample Y, of the basis Q and of U.
The global power iteration of ``rsvd_incore`` (rsvd.py:126-141) /
``rsvd_naive_ooc`` (rsvd.py:218-284) then needs exactly these exchanges:

  * Z = sum_g A_g^T Y_g            (n x l)   all-reduce, once per power pass
  * G = sum_g Y_g^T Y_g            (l x l)   all-reduce, per CholQR pass
  * C = sum_g Q_g^T W_g            (k x c)   all-reduce, completion (rare)
  * B^T = sum_g A_g^T Q_g          (n x l)   all-reduce, once
  * column argmax of U             (l)       all-gather, for the signs

The shard is either resident in HBM (a torch CUDA tensor) or host-resident
(``HostShard``: BASELINE config 4, each rank streams its own row panels over
its own PCIe link through the panel streamer, one pass per power step --
``brsvd_stream_rows_pass`` forms Y_i = A_i X and accumulates A_i^T Y_i from
the same panel load, so the decomposition costs q + 2 passes over A).
Everything else is local (the A-streaming products) or replicated and
bit-identical on every rank (the l x l factorisations, the small SVD), so U
stays row-sharded and sigma, Vt are replicated.  The stage operations come
from an ``ops`` object: ``GpuOps`` calls the C ABI (tcgen05 products, fp64
Gram/Cholesky kernels, Jacobi small SVD) on the local GPU; the tests run the
same driver with numpy operations over the gloo backend.
"""

import ctypes
import math

import numpy as np

from . import _lib
from .kernels import SvdFactors

_EPS = {np.dtype(np.float64): 2.220446049250313e-16,
        np.dtype(np.float32): 1.1920928955078125e-07}


# ---------------------------------------------------------------------------
class TorchComm:
    """Collectives over torch.distributed (NCCL for CUDA tensors; host
    round-trip for gloo).  World size 1 needs no process group."""

    def __init__(self, group=None):
        import torch.distributed as dist
        self.dist = dist
        self.group = group
        self.active = dist.is_available() and dist.is_initialized()
        self.world = dist.get_world_size(group) if self.active else 1
        self.rank = dist.get_rank(group) if self.active else 0
        self.backend = dist.get_backend(group) if self.active else None

    def _as_tensor(self, x):
        """A contiguous tensor sharing x's memory (column-major views are
        transposed, which leaves the element-wise reductions unchanged)."""
        import torch
        if isinstance(x, np.ndarray):
            return torch.from_numpy(x if x.flags.c_contiguous else x.T)
        return x if x.is_contiguous() else x.t()

    def allreduce_sum(self, x):
        if self.world == 1:
            return x
        t = self._as_tensor(x)
        if t.is_cuda and self.backend != "nccl":
            h = t.cpu()
            self.dist.all_reduce(h, group=self.group)
            t.copy_(h)
        else:
            self.dist.all_reduce(t, group=self.group)
        return x

    def allreduce_max(self, value):
        if self.world == 1:
            return value
        import torch
        dev = "cuda" if self.backend == "nccl" else "cpu"
        t = torch.tensor([value], dtype=torch.float64, device=dev)
        self.dist.all_reduce(t, op=self.dist.ReduceOp.MAX, group=self.group)
        return float(t.item())

    def allgather_array(self, arr):
        """All-gather of a small float64 array (one tensor collective)."""
        if self.world == 1:
            return [np.asarray(arr)]
        import torch
        dev = "cuda" if self.backend == "nccl" else "cpu"
        t = torch.as_tensor(np.ascontiguousarray(arr, dtype=np.float64), device=dev)
        out = [torch.empty_like(t) for _ in range(self.world)]
        self.dist.all_gather(out, t, group=self.group)
        return [o.cpu().numpy() for o in out]

    def allgather_obj(self, obj):
        if self.world == 1:
            return [obj]
        out = [None] * self.world
        self.dist.all_gather_object(out, obj, group=self.group)
        return out


class NcclComm:
    """Collectives on the library's own NCCL communicator
    (brsvd_ctx_attach_nccl): they run on the context's stream, in order with
    the kernels that produce and consume them, and fail as BRSVD_ERR_NCCL.
    The 128-byte unique id travels once through torch.distributed (any
    backend, plumbing only); world size 1 needs no process group.  Same
    interface as TorchComm for rsvd_sharded."""

    def __init__(self, ops, group=None):
        import torch
        import torch.distributed as dist
        self.ops = ops
        self.torch = torch
        active = dist.is_available() and dist.is_initialized()
        self.world = dist.get_world_size(group) if active else 1
        self.rank = dist.get_rank(group) if active else 0
        lib = _lib.load_library()
        uid = ctypes.create_string_buffer(128)
        if self.rank == 0:
            _lib.check(lib.brsvd_nccl_unique_id(uid))
        if self.world > 1:
            box = [bytes(uid.raw) if self.rank == 0 else None]
            dist.broadcast_object_list(box, src=0, group=group)
            uid = ctypes.create_string_buffer(box[0], 128)
        _lib.check(lib.brsvd_ctx_attach_nccl(ops.ctx.handle, uid, self.world, self.rank))
        self.lib = lib

    def _dense(self, x):
        """A contiguous CUDA tensor sharing x's storage (column-major views
        are transposed: element-wise reductions do not care)."""
        t = x if x.is_contiguous() else x.t()
        if not t.is_contiguous():
            raise ValueError("collective operand must be dense")
        return t

    def allreduce_sum(self, x):
        t = self._dense(x)
        self.ops._sync_stream()
        code = 1 if t.dtype == self.torch.float64 else 2
        _lib.check(self.lib.brsvd_allreduce(self.ops.ctx.handle, ctypes.c_void_p(t.data_ptr()),
                                            t.numel(), code, 0))
        return x

    def allreduce_max(self, value):
        t = self.torch.tensor([float(value)], dtype=self.torch.float64,
                              device=self.ops.device)
        self.ops._sync_stream()
        _lib.check(self.lib.brsvd_allreduce(self.ops.ctx.handle, ctypes.c_void_p(t.data_ptr()),
                                            1, 1, 2))
        return float(t.item())

    def allgather_array(self, arr):
        a = np.ascontiguousarray(arr, dtype=np.float64)
        send = self.torch.as_tensor(a, device=self.ops.device)
        recv = self.torch.empty((self.world,) + a.shape, dtype=self.torch.float64,
                                device=self.ops.device)
        self.ops._sync_stream()
        _lib.check(self.lib.brsvd_allgather(self.ops.ctx.handle,
                                            ctypes.c_void_p(send.data_ptr()),
                                            ctypes.c_void_p(recv.data_ptr()), send.numel(), 1))
        out = recv.cpu().numpy()
        return [out[r] for r in range(self.world)]


# ---------------------------------------------------------------------------
class HostShard:
    """This rank's row shard A[r0:r1, :] held in host memory (pinned for
    overlapped DMA, e.g. a numpy view of ``torch.empty(..., pin_memory=True)``),
    streamed to the GPU in row panels of ``panel`` rows through ``nbuf``
    device buffers once per pass (store.py:165-175 reads a column block per
    pass the same way; here the unit is a row panel of the rank's shard).
    C-ordered or Fortran-ordered arrays are accepted."""

    def __init__(self, a, panel=None, nbuf=3):
        a = np.asarray(a)
        if a.ndim != 2:
            from .kernels import ShapeError
            raise ShapeError(f"expected a 2-D shard, got shape {a.shape}")
        if a.dtype not in (np.float32, np.float64):
            a = a.astype(np.float64)
        if not (a.flags.c_contiguous or a.flags.f_contiguous):
            a = np.ascontiguousarray(a)
        self.a = a
        self.shape = a.shape
        self.dtype = a.dtype
        if panel is None:   # ~512 MiB panels
            panel = max(1, (512 << 20) // max(1, a.shape[1] * a.itemsize))
        self.panel = int(panel)
        self.nbuf = int(nbuf)
        self.passes = 0
        self.pass_ms = []

    @property
    def nbytes(self):
        return self.a.nbytes


# ---------------------------------------------------------------------------
def _cm_empty(rows, cols, dtype, device):
    """Column-major (rows x cols) torch tensor (storage = (cols, rows))."""
    import torch
    return torch.empty((cols, rows), dtype=dtype, device=device).t()


def _ld(t):
    return max(t.stride(1), 1)


def _code(t):
    import torch
    return _lib.F64 if t.dtype == torch.float64 else _lib.F32


def _vp(t):
    return ctypes.c_void_p(t.data_ptr())


class GpuOps:
    """Local stage operations on torch CUDA tensors through the C ABI.

    Tall-skinny matrices are column-major torch views (shape (rows, cols),
    stride (1, rows)); A may be row- or column-major.
    """

    def __init__(self, device=None):
        import torch
        self.torch = torch
        self.device = torch.device("cuda", torch.cuda.current_device()
                                   if device is None else device)
        self.ctx = _lib.context(self.device.index)
        self.lib = _lib.load_library()

    def _sync_stream(self):
        self.ctx.set_stream(self.torch.cuda.current_stream(self.device).cuda_stream)

    def asarray(self, x, dtype):
        t = self.torch.as_tensor(np.asarray(x) if not hasattr(x, "data_ptr") else x,
                                 device=self.device, dtype=dtype)
        out = _cm_empty(t.shape[0], t.shape[1], dtype, self.device)
        out.copy_(t)
        return out

    def dtype_of(self, A):
        return A.dtype

    def absmax(self, A):
        """(row maxima, column maxima) of |A| for the fp16-split products
        (brsvd_absmax), once per decomposition; None for fp64 data."""
        from ._arrays import DeviceMatrix
        if A.dtype != self.torch.float32:
            return None
        self._sync_stream()
        mat = DeviceMatrix(A)
        m, n = mat.shape
        rmax = self.torch.empty(m, dtype=self.torch.float32, device=self.device)
        cmax = self.torch.empty(n, dtype=self.torch.float32, device=self.device)
        _lib.check(self.lib.brsvd_absmax(self.ctx.handle, mat.ptr, m, n, mat.ld, mat.code,
                                         mat.layout, _vp(rmax), _vp(cmax)))
        return rmax, cmax

    def product(self, A, X, trans, amax=None):
        from ._arrays import DeviceMatrix
        self._sync_stream()
        mat = DeviceMatrix(A)
        m, n = mat.shape
        rows = n if trans else m
        l = X.shape[1]
        C = _cm_empty(rows, l, A.dtype, self.device)
        scale = None if amax is None else _vp(amax[1] if trans else amax[0])
        _lib.check(self.lib.brsvd_sketch_product_scaled(
            self.ctx.handle, mat.ptr, m, n, mat.ld, mat.code, mat.layout, int(trans),
            _vp(X), _ld(X), l, _vp(C), rows, scale))
        return C

    def gram(self, X, W=None):
        self._sync_stream()
        k1 = X.shape[1]
        k2 = W.shape[1] if W is not None else k1
        G = _cm_empty(k1, k2, self.torch.float64, self.device)
        _lib.check(self.lib.brsvd_gram(
            self.ctx.handle, _vp(X), X.shape[0], k1, _ld(X), _code(X),
            _vp(W) if W is not None else None, k2, _ld(W) if W is not None else 1, _vp(G)))
        return G

    def chol_basis(self, G, shift=0.0, col_drop=0.0, rank_tol=0.0, drop_ratio=0.0):
        self._sync_stream()
        l = G.shape[0]
        Gc = G.clone()
        T = _cm_empty(l, l, self.torch.float64, self.device)
        kept, rank = ctypes.c_int32(), ctypes.c_int32()
        _lib.check(self.lib.brsvd_chol_basis(
            self.ctx.handle, _vp(Gc), l, ctypes.c_double(shift), ctypes.c_double(col_drop),
            ctypes.c_double(rank_tol), ctypes.c_double(drop_ratio), _vp(T),
            ctypes.byref(kept), ctypes.byref(rank)))
        return T, kept.value, rank.value

    def apply(self, X, T, out_dtype, out=None, alpha=1.0, beta=0.0):
        self._sync_stream()
        r, k = X.shape
        kt = T.shape[1]
        if out is None:
            out = _cm_empty(r, kt, out_dtype, self.device)
        Tc = T if T.stride(0) == 1 and T.stride(1) == k else T.t().contiguous().t()
        _lib.check(self.lib.brsvd_apply(
            self.ctx.handle, _vp(X), r, k, _ld(X), _code(X), _vp(Tc), kt, _vp(out), _ld(out),
            _code(out), ctypes.c_double(alpha), ctypes.c_double(beta)))
        return out

    def normalize(self, Z):
        self._sync_stream()
        out = _cm_empty(Z.shape[0], Z.shape[1], Z.dtype, self.device)
        _lib.check(self.lib.brsvd_normalize(self.ctx.handle, _vp(Z), Z.shape[0], Z.shape[1],
                                            _ld(Z), _code(Z), _vp(out), _ld(out)))
        return out

    def gaussian(self, rows, cols, seed, stream, row_offset, dtype):
        self._sync_stream()
        out = _cm_empty(rows, cols, dtype, self.device)
        _lib.check(self.lib.brsvd_gaussian(
            self.ctx.handle, _vp(out), rows, cols, rows, _code(out),
            ctypes.c_uint64(seed & (2 ** 64 - 1)), ctypes.c_uint64(stream & (2 ** 64 - 1)),
            int(row_offset)))
        return out

    def small_svd(self, Bt):
        self._sync_stream()
        n, l = Bt.shape
        W = _cm_empty(l, l, Bt.dtype, self.device)
        sigma = self.torch.empty(l, dtype=Bt.dtype, device=self.device)
        Vt = self.torch.empty((l, n), dtype=Bt.dtype, device=self.device)
        rank = ctypes.c_int32()
        _lib.check(self.lib.brsvd_small_svd(
            self.ctx.handle, _vp(Bt), n, l, _ld(Bt), _code(Bt), _lib.DEVICE, _vp(W),
            _vp(sigma), _vp(Vt), ctypes.byref(rank)))
        return W.double(), sigma, Vt, rank.value

    def colmax(self, U, row_offset):
        self._sync_stream()
        l = U.shape[1]
        vals = np.empty(l, dtype=np.float64)
        idx = np.empty(l, dtype=np.int64)
        _lib.check(self.lib.brsvd_colmax(self.ctx.handle, _vp(U), U.shape[0], l, _ld(U),
                                         _code(U), int(row_offset),
                                         ctypes.c_void_p(vals.ctypes.data),
                                         ctypes.c_void_p(idx.ctypes.data)))
        return vals, idx

    def colmax_entries(self, U, row_offset):
        """(3, l) float64: per column max |u|, its global row, the signed u
        there (brsvd_colmax_entries: one kernel, one D2H copy)."""
        self._sync_stream()
        l = U.shape[1]
        out = np.empty(3 * l, dtype=np.float64)
        _lib.check(self.lib.brsvd_colmax_entries(self.ctx.handle, _vp(U), U.shape[0], l, _ld(U),
                                                 _code(U), int(row_offset),
                                                 ctypes.c_void_p(out.ctypes.data)))
        return out.reshape(3, l)

    def stream_pass(self, shard, X, Y=None, want_z=False):
        """One pass of the host-resident shard through the panel streamer
        (brsvd_stream_rows_pass): Y = A X when X is given (else Y is an
        input), and the fp64 Z = A^T Y when want_z.  Returns (Y, Z)."""
        self._sync_stream()
        a = shard.a
        m, n = a.shape
        layout = _lib.ROW_MAJOR if a.flags.c_contiguous else _lib.COL_MAJOR
        lda = n if layout == _lib.ROW_MAJOR else m
        tdt = self.torch.float64 if a.dtype == np.float64 else self.torch.float32
        l = X.shape[1] if X is not None else Y.shape[1]
        if Y is None:
            Y = _cm_empty(m, l, tdt, self.device)
        Z = _cm_empty(n, l, self.torch.float64, self.device) if want_z else None
        ms = ctypes.c_double()
        _lib.check(self.lib.brsvd_stream_rows_pass(
            self.ctx.handle, ctypes.c_void_p(a.ctypes.data), m, n, lda, _lib.dtype_code(a.dtype),
            layout, _vp(X) if X is not None else None, _ld(X) if X is not None else 1, l,
            _vp(Y), _ld(Y), _vp(Z) if Z is not None else None, _ld(Z) if Z is not None else 1,
            shard.panel, shard.nbuf, ctypes.byref(ms)))
        shard.passes += 1
        shard.pass_ms.append(ms.value)
        return Y, Z

    def normalize_f64(self, Z, dtype, T=None):
        """Basis change of an fp64 Z (brsvd_normalize_f64) in the data's dtype;
        with T (device l x l fp64 buffer) also returns the power-of-two scale s
        of Zout = (s Z) T."""
        self._sync_stream()
        out = _cm_empty(Z.shape[0], Z.shape[1], dtype, self.device)
        sc = ctypes.c_double(1.0)
        _lib.check(self.lib.brsvd_normalize_f64(self.ctx.handle, _vp(Z), Z.shape[0], Z.shape[1],
                                                _ld(Z), _code(out), _vp(out), _ld(out),
                                                None if T is None else _vp(T),
                                                ctypes.byref(sc)))
        return out if T is None else (out, sc.value)

    def normalize_t(self, Z, T):
        """brsvd_normalize writing the applied transform into T (device l x l
        fp64): Zout = Z T."""
        self._sync_stream()
        out = _cm_empty(Z.shape[0], Z.shape[1], Z.dtype, self.device)
        _lib.check(self.lib.brsvd_normalize_t(self.ctx.handle, _vp(Z), Z.shape[0], Z.shape[1],
                                              _ld(Z), _code(Z), _vp(out), _ld(out), _vp(T)))
        return out

    def transform_buffers(self, q, l):
        return self.torch.empty((q, l, l), dtype=self.torch.float64, device=self.device)

    def unnormalised_peak(self, Y, Ts, zfac):
        """max |Y (prod zfac_i T_i)^-1| over this rank's rows (brsvd_unnormalised_peak)."""
        self._sync_stream()
        z = np.ascontiguousarray(zfac, dtype=np.float64)
        out = ctypes.c_double()
        Yc = Y if _ld(Y) == Y.shape[0] else Y.t().contiguous().t()
        _lib.check(self.lib.brsvd_unnormalised_peak(
            self.ctx.handle, _vp(Yc), Y.shape[0], Y.shape[1], _code(Y), len(z), _vp(Ts),
            ctypes.c_void_p(z.ctypes.data), ctypes.byref(out)))
        return out.value

    def scale_cols(self, X, scale):
        self._sync_stream()
        s = np.ascontiguousarray(scale, dtype=np.float64)
        _lib.check(self.lib.brsvd_scale_cols(self.ctx.handle, _vp(X), X.shape[0], X.shape[1],
                                             _ld(X), _code(X),
                                             ctypes.c_void_p(s.ctypes.data)))
        return X

    def hstack(self, a, b):
        out = _cm_empty(a.shape[0], a.shape[1] + b.shape[1], a.dtype, self.device)
        out[:, :a.shape[1]] = a
        out[:, a.shape[1]:] = b
        return out

    def cols(self, X, k):
        return X[:, :k]

    def cast(self, X, dtype):
        out = _cm_empty(X.shape[0], X.shape[1], dtype, self.device)
        out.copy_(X)
        return out


# ---------------------------------------------------------------------------
def _orth_sharded(Y, ops, comm, eps_data, row_offset, m_total, seed):
    """Rank-revealing CholQR2 of the row-sharded Y (orth.cuh orth_full,
    level 1 + completion) with all-reduced Grams."""
    l = Y.shape[1]
    G = comm.allreduce_sum(ops.gram(Y))
    T, kept, rank_ref = ops.chol_basis(G, 0.0, 4.0 * l * eps_data, l * eps_data, 1e-12)
    if eps_data > 1e-10:
        # fp32 data (orth_full_f32): fp32 basis, the dropped directions
        # completed by Gaussian columns inside the second CholQR pass
        dt = ops.dtype_of(Y)
        Q1 = ops.apply(Y, ops.cols(T, kept), dt) if kept > 0 else None
        if kept < l:
            W = ops.gaussian(Y.shape[0], l - kept, seed, 0x636f6d706c657465, row_offset, dt)
            Q1 = W if Q1 is None else ops.hstack(Q1, W)
        G2 = comm.allreduce_sum(ops.gram(Q1))
        T2, _, _ = ops.chol_basis(G2)
        return ops.apply(Q1, T2, dt), min(rank_ref, kept)
    f64 = ops.torch.float64 if hasattr(ops, "torch") else np.float64
    Q = None
    if kept > 0:
        Q1 = ops.apply(Y, ops.cols(T, kept), f64)
        G2 = comm.allreduce_sum(ops.gram(Q1))
        T2, _, _ = ops.chol_basis(G2)
        Q = ops.apply(Q1, ops.cols(T2, kept), f64)
    if kept < l:
        cnt = l - kept
        W = ops.gaussian(Y.shape[0], cnt, seed, 0x636f6d706c657465, row_offset, f64)
        if Q is not None:
            for _ in range(2):
                C = comm.allreduce_sum(ops.gram(Q, W))
                W = ops.apply(Q, C, f64, out=W, alpha=-1.0, beta=1.0)
        for _ in range(2):
            Gw = comm.allreduce_sum(ops.gram(W))
            Tw, _, _ = ops.chol_basis(Gw)
            W = ops.apply(W, Tw, f64)
        Q = W if Q is None else ops.hstack(Q, W)
    return Q, min(rank_ref, kept)


def _sign_flips(cands, l):
    """_fix_signs (rsvd.py:105-115) over the global rows: per column, the
    first row (lowest global index) of the largest |u| decides; cands are the
    ranks' (3, l) [max |u|, global row, signed u] arrays."""
    signs = np.ones(l)
    for j in range(l):
        best = None
        for c in cands:
            v, i, e = float(c[0, j]), float(c[1, j]), float(c[2, j])
            if v != v:
                v = np.inf
            if best is None or v > best[0] or (v == best[0] and i < best[1]):
                best = (v, i, e)
        signs[j] = -1.0 if best[2] < 0 else 1.0
    return signs


def rsvd_sharded(A_local, cfg, row_offset, m_total, comm=None, ops=None, omega=None):
    """Randomized SVD of the row-sharded matrix whose rows
    [row_offset, row_offset + A_local.shape[0]) this rank holds.

    ``A_local`` is resident (torch CUDA tensor; numpy with the test ops) or a
    ``HostShard`` streamed from host memory (q + 2 passes over PCIe).
    Returns (factors, info): factors.U holds this rank's rows of U;
    sigma and Vt are replicated.  Same semantics (global power iteration) and
    validation as rsvd_incore (rsvd.py:126-141) / rsvd_naive_ooc
    (rsvd.py:218-284).
    """
    comm = comm or TorchComm()
    ops = ops or GpuOps()
    row_offset, m_total = int(row_offset), int(m_total)
    streamed = isinstance(A_local, HostShard)
    m_loc, n = A_local.shape
    cfg.validate(m_total, n)
    k, p, q = cfg.target_rank, cfg.oversampling, cfg.power_exponent
    l = k + p
    if streamed:
        npdt = np.dtype(A_local.dtype)
        dtype = (ops.torch.float64 if npdt == np.float64 else ops.torch.float32) \
            if hasattr(ops, "torch") else npdt
    else:
        dtype = ops.dtype_of(A_local)
        npdt = np.dtype(np.float64) if str(dtype).endswith("float64") else np.dtype(np.float32)
    eps_data = _EPS[npdt]
    seed = int(cfg.master_seed)
    X = ops.asarray(omega, dtype) if omega is not None else ops.gaussian(n, l, seed, 0, 0, dtype)
    # the applied basis changes, for the exact overflow guard (Cholesky route,
    # l <= 320 as pipeline.cuh): Zn_i = (zfac_i Z_i) T_i
    track = q > 0 and l <= 320 and hasattr(ops, "unnormalised_peak")
    Ts = ops.transform_buffers(q, l) if track else None
    zfac = []
    if streamed:
        def sample(Xs, want_z):
            return ops.stream_pass(A_local, Xs, None, want_z)

        def basis(Z, it):
            if not track:
                return ops.normalize_f64(Z, dtype)
            Zn, sc = ops.normalize_f64(Z, dtype, Ts[it])
            zfac.append(sc)
            return Zn
    else:
        amax = ops.absmax(A_local) if hasattr(ops, "absmax") else None

        def sample(Xs, want_z):
            Ys = ops.product(A_local, Xs, False, amax)
            return Ys, (ops.product(A_local, Ys, True, amax) if want_z else None)

        def basis(Z, it):
            if not track:
                return ops.normalize(Z)
            zfac.append(1.0)
            return ops.normalize_t(Z, Ts[it])
    Y, Zp = sample(X, q > 0)
    vals = ops.colmax_entries(Y, row_offset)[0]
    bad = not np.all(np.isfinite(vals)) or np.any(vals < 0)
    peak0 = comm.allreduce_max(float(np.max(vals)) if vals.size else 0.0)
    bad = comm.allreduce_max(1.0 if bad else 0.0) > 0
    if bad:
        raise FloatingPointError("sample matrix is not finite; the overflow guard fires")
    for it in range(q):
        Z = comm.allreduce_sum(Zp)
        Y, Zp = sample(basis(Z, it), it < q - 1)
    Q, rank_y = _orth_sharded(Y, ops, comm, eps_data, row_offset, m_total, seed ^ 0x7153)
    Qd = ops.cast(Q, dtype)
    if streamed:
        _, Bt64 = ops.stream_pass(A_local, None, Qd, True)
        Bt = ops.cast(comm.allreduce_sum(Bt64), dtype)
    else:
        Bt = comm.allreduce_sum(ops.product(A_local, Qd, True, amax))
    W, sigma, Vt, rank_b = ops.small_svd(Bt)
    U = ops.apply(Q, W, dtype)
    signs = _sign_flips(comm.allgather_array(ops.colmax_entries(U, row_offset)), l)
    ops.scale_cols(U, signs)
    ops.scale_cols(Vt.t() if hasattr(Vt, "t") and not isinstance(Vt, np.ndarray) else Vt.T,
                   signs)
    s0 = float(sigma[0])
    lim = math.log10(0.01 * np.finfo(npdt).max)
    if not math.isfinite(s0):   # as pipeline.cuh: a non-finite sigma_1 is an overflow
        raise FloatingPointError("sample matrix is not finite; the overflow guard fires")
    # _check_overflow (rsvd.py:84-91) on the reference's unnormalised sample:
    # far below the threshold the bound max|A Omega| sqrt(m) s_1^(2q) settles
    # it; near or above it the peak is formed exactly from this rank's rows
    # and the kept transforms (one all-reduce max), as pipeline.cuh does
    log_peak = (math.log10(peak0) + 2 * q * math.log10(s0)) if peak0 > 0 and s0 > 0 else -400.0
    if q == 0:
        over = log_peak > lim
    elif log_peak + 0.5 * math.log10(m_total) + 0.05 <= lim:
        over = False
    elif track:
        pk = comm.allreduce_max(ops.unnormalised_peak(Y, Ts, zfac))
        log_peak = math.log10(pk) if pk > 0 else -400.0
        over = not (pk <= 0.01 * float(np.finfo(npdt).max))
    else:
        over = log_peak > lim
    if over:
        raise FloatingPointError("sample matrix magnitude exceeds the overflow guard")
    info = {"rank_y": rank_y, "rank_b": rank_b, "max_abs_y0": peak0, "log10_peak": log_peak}
    if streamed:
        info.update(passes=A_local.passes, pass_ms=list(A_local.pass_ms),
                    h2d_bytes=A_local.passes * A_local.nbytes)
    return SvdFactors(U=U, sigma=sigma, Vt=Vt, target_rank=k, effective_l=l), info
