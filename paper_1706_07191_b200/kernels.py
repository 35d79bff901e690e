"""Dense building blocks of the hot path, executed on the B200.

Drop-in for the reference module ``blocksvd.kernels`` (kernels.py): same
names, argument meaning, return types and exceptions.  The arithmetic runs in
the CUDA library behind include/brsvd.h; this module only marshals operands.

Deltas from the reference (documented in DESIGN.md):
  * ``gaussian_matrix`` uses a counter-based Philox4x32 + Box-Muller stream on
    the GPU.  Entries are a pure function of (seed, stream, row, col) as in
    kernels.py:98-118, but the values differ from numpy's ziggurat stream.
    Parity runs inject the reference's Omega instead (rsvd_incore(omega=...)).
  * ``tsqr_factor`` returns an orthonormal Q and a square R with Y = Q R; R is
    not triangular (the basis comes from a rank-revealing Gram
    eigendecomposition, not Householder reflections).  ``block_rows`` is
    accepted for signature compatibility; the GPU algorithm has no tree.
"""

import ctypes
import warnings
from dataclasses import dataclass

import numpy as np

from . import _lib
from ._arrays import HostMatrix

__all__ = [
    "ShapeError",
    "RankDeficiencyWarning",
    "SvdFactors",
    "gaussian_matrix",
    "tsqr",
    "tsqr_factor",
    "small_svd",
]


class ShapeError(ValueError):
    """Operand dimensions do not conform (kernels.py:27-28)."""


class RankDeficiencyWarning(UserWarning):
    """Input to a factorization is numerically rank deficient (kernels.py:31-39).

    The detected numerical rank is available as ``detected_rank``.
    """

    def __init__(self, message, detected_rank):
        super().__init__(message)
        self.detected_rank = detected_rank


@dataclass
class SvdFactors:
    """Approximate SVD triple U * diag(sigma) * Vt (kernels.py:42-66)."""

    U: object
    sigma: object
    Vt: object
    target_rank: int
    effective_l: int

    def truncate(self, rank=None):
        r = self.target_rank if rank is None else rank
        if r > self.effective_l:
            raise ValueError(f"rank {r} exceeds computed width {self.effective_l}")
        return SvdFactors(self.U[:, :r], self.sigma[:r], self.Vt[:r, :], r, r)

    def compose(self):
        return (self.U * self.sigma) @ self.Vt


def warn_rank(rank, l):
    if rank < l:
        warnings.warn(RankDeficiencyWarning(
            f"input has numerical rank {rank} < {l}", rank), stacklevel=3)


def gaussian_matrix(rows, cols, master_seed, stream_index=0, row_offset=0,
                    dtype=np.float64):
    """Seeded i.i.d. standard-normal matrix generated on the GPU.

    Entries are a pure function of (master_seed, stream_index,
    row_offset + row, column), so a block generated with the matching
    ``row_offset`` is bit-identical to the corresponding slice of the full
    matrix (the property kernels.py:98-118 guarantees).
    """
    if rows < 1 or cols < 1:
        raise ShapeError(f"gaussian_matrix needs positive shape, got {rows}x{cols}")
    import torch
    dt = np.dtype(dtype)
    code = _lib.dtype_code(dt)
    ctx = _lib.context()
    tdt = torch.float64 if code == _lib.F64 else torch.float32
    dev = torch.empty((cols, rows), dtype=tdt, device=f"cuda:{ctx.device}")
    _lib.check(_lib.load_library().brsvd_gaussian(
        ctx.handle, ctypes.c_void_p(dev.data_ptr()), rows, cols, rows, code,
        ctypes.c_uint64(int(master_seed) & (2 ** 64 - 1)),
        ctypes.c_uint64(int(stream_index) & (2 ** 64 - 1)), int(row_offset)))
    return np.asfortranarray(dev.cpu().numpy().T)


def tsqr_factor(y, block_rows=None):
    """Orthonormal Q (m x l) and R (l x l) with y = Q R (kernels.py:139-164).

    Rank deficiency is tolerated: columns of Q stay orthonormal and a
    RankDeficiencyWarning reports the detected numerical rank.
    """
    y = np.asarray(y)
    if y.ndim != 2:
        raise ShapeError("tsqr expects a 2-D array")
    m, l = y.shape
    if m < l:
        raise ShapeError(f"tsqr requires rows >= cols, got {m}x{l}")
    hm = HostMatrix(np.asfortranarray(y), "y")
    q = np.empty((m, l), dtype=hm.dtype, order="F")
    r = np.empty((l, l), dtype=hm.dtype, order="F")
    rank = ctypes.c_int32()
    ctx = _lib.context()
    _lib.check(_lib.load_library().brsvd_tsqr(
        ctx.handle, hm.ptr, m, l, hm.ld, hm.code, _lib.HOST,
        ctypes.c_void_p(q.ctypes.data), ctypes.c_void_p(r.ctypes.data),
        ctypes.byref(rank)))
    warn_rank(rank.value, l)
    return q, r


def tsqr(y, block_rows=None):
    """Orthonormal basis of range(y); see tsqr_factor."""
    q, _ = tsqr_factor(y, block_rows)
    return q


def small_svd(b):
    """SVD of a short-fat l-by-n matrix (kernels.py:173-188).

    b.T = Qb R (rank-revealing orthonormal basis), R.T = W s Zt (one-sided
    Jacobi), b = W s (Zt Qb.T).
    """
    b = np.asarray(b)
    if b.ndim != 2:
        raise ShapeError("small_svd expects a 2-D array")
    l, n = b.shape
    if l > n:
        raise ShapeError(f"small_svd requires rows <= cols, got {l}x{n}")
    hb = HostMatrix(np.ascontiguousarray(b), "b")   # row-major l x n == Bt col-major
    w = np.empty((l, l), dtype=hb.dtype, order="F")
    sigma = np.empty(l, dtype=hb.dtype)
    vt = np.empty((l, n), dtype=hb.dtype, order="C")
    rank = ctypes.c_int32()
    ctx = _lib.context()
    _lib.check(_lib.load_library().brsvd_small_svd(
        ctx.handle, hb.ptr, n, l, n, hb.code, _lib.HOST,
        ctypes.c_void_p(w.ctypes.data), ctypes.c_void_p(sigma.ctypes.data),
        ctypes.c_void_p(vt.ctypes.data), ctypes.byref(rank)))
    warn_rank(rank.value, l)
    return SvdFactors(U=w, sigma=sigma, Vt=vt, target_rank=l, effective_l=l)
