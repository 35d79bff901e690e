"""CPU oracle for the BRSVD hot path: a numpy restatement of the reference.

TEST INFRASTRUCTURE ONLY.  This module is the checker: it may be imported by
tests/, by __graft_entry__.smoke() and by bench.py's ``cpu_baseline`` /
``--impl reference`` legs, and never by the product package
(paper_1706_07191_b200), which has no CPU path.

It restates, function by function, the algorithm of the reference package
``blocksvd`` (/root/reference/pkg/src/blocksvd), whose arithmetic lives in the
third-party dependency numpy (unpinned, ``numpy>=1.24``,
/root/reference/pkg/pyproject.toml:10; this image has numpy 2.3.5 with
OpenBLAS 0.3.30): matrix products are ``@`` (BLAS gemm), QR is
``np.linalg.qr`` (LAPACK geqrf/orgqr), the small SVD is ``np.linalg.svd``
(LAPACK gesdd), and the Gaussian sketch is numpy's Philox4x64-10 bit
generator with its ziggurat normal transform.

Parity pinning: tests/test_oracle_golden.py checks every function here
against tests/golden/*.npz, which oracle/make_golden.py produced by running the
reference package itself in the build container.
"""

import numpy as np


# --- kernels.py ---------------------------------------------------------------

def normal_sketch(rows, cols, seed, stream=0, row_offset=0, dtype=np.float64):
    """Gaussian sketch, one independent Philox stream per global row.

    kernels.py:90-95: key = [seed, stream], counter = row << 192 (the row
    index occupies the top word of the 256-bit counter);
    kernels.py:112-118: each row is ``standard_normal(cols, dtype)`` of its
    own generator, stored into a Fortran-ordered matrix.
    """
    if rows < 1 or cols < 1:
        raise ValueError(f"gaussian_matrix needs positive shape, got {rows}x{cols}")
    out = np.empty((rows, cols), dtype=dtype, order="F")
    key = np.array([seed, stream], dtype=np.uint64)
    for i in range(rows):
        gen = np.random.Generator(np.random.Philox(key=key, counter=(row_offset + i) << 192))
        out[i] = gen.standard_normal(cols, dtype=dtype)
    return out


def _tree_qr(y, leaf):
    """Recursive row-block Householder QR (kernels.py:121-136).

    Split at the largest multiple of ``leaf`` not exceeding half the blocks,
    factor both halves, then QR the stacked R factors.
    """
    m, l = y.shape
    if m <= leaf:
        return np.linalg.qr(y, mode="reduced")
    blocks = -(-m // leaf)
    cut = (blocks // 2) * leaf
    qa, ra = _tree_qr(y[:cut], leaf)
    qb, rb = _tree_qr(y[cut:], leaf)
    qs, r = np.linalg.qr(np.vstack([ra, rb]), mode="reduced")
    return np.vstack([qa @ qs[:l], qb @ qs[l:]]), r


def orthonormal_range(y, block_rows=None):
    """(Q, R, rank) of the tall-skinny QR (kernels.py:139-164).

    Leaf height defaults to 64*l, never below 2*l; the numerical rank counts
    |diag R| above l * eps * ||y||_F.
    """
    m, l = y.shape
    if m < l:
        raise ValueError(f"tsqr requires rows >= cols, got {m}x{l}")
    leaf = max(64 * l if block_rows is None else block_rows, 2 * l)
    q, r = _tree_qr(y, leaf)
    cut = l * np.finfo(y.dtype).eps * np.linalg.norm(y)
    rank = int(np.count_nonzero(np.abs(np.diag(r)) > cut))
    return q, r, rank


def core_svd(b):
    """SVD of a short-fat b (kernels.py:173-188): QR(b^T) then LAPACK SVD of
    the small triangular factor; returns (W, s, Vt, rank_of_b)."""
    l, n = b.shape
    if l > n:
        raise ValueError(f"small_svd requires rows <= cols, got {l}x{n}")
    qb, r, rank = orthonormal_range(np.ascontiguousarray(b.T))
    w, s, zt = np.linalg.svd(r.T, full_matrices=False)
    return w, s, zt @ qb.T, rank


# --- rsvd.py -------------------------------------------------------------------

def canonical_signs(u, vt):
    """Largest-|.| entry of each left vector made non-negative (rsvd.py:105-115).
    Returns new arrays."""
    u = u.copy()
    vt = vt.copy()
    pivot = np.argmax(np.abs(u), axis=0)
    sgn = np.sign(u[pivot, np.arange(u.shape[1])])
    sgn[sgn == 0] = 1.0
    return u * sgn, vt * sgn[:, None]


def power_sample(a, omega, q):
    """(A A^T)^q A Omega evaluated right to left (rsvd.py:94-102)."""
    y = a @ omega
    for _ in range(q):
        y = a @ (a.T @ y)
    return y


def overflow_peak(y):
    """Peak magnitude and whether it trips the guard (rsvd.py:84-91)."""
    peak = np.max(np.abs(y))
    return peak, (not np.isfinite(peak)) or peak > 0.01 * np.finfo(y.dtype).max


def randomized_svd(a, k, p=10, q=0, seed=0, omega=None):
    """rsvd_incore (rsvd.py:126-141) with its helpers _finish (rsvd.py:118-123).

    Returns dict(U, sigma, Vt, omega, rank_y, rank_b, peak, overflow).
    """
    m, n = a.shape
    l = k + p
    if omega is None:
        omega = normal_sketch(n, l, seed, 0, dtype=a.dtype)
    y = power_sample(a, omega, q)
    peak, over = overflow_peak(y)
    if over:
        return dict(overflow=True, peak=peak)
    qy, _, rank_y = orthonormal_range(y)
    w, s, vt, rank_b = core_svd(qy.T @ a)
    u, vt = canonical_signs(qy @ w, vt)
    return dict(U=u, sigma=s, Vt=vt, omega=omega, rank_y=rank_y, rank_b=rank_b,
                peak=peak, overflow=False)


def column_blocks(n, s):
    width = -(-n // s)
    return [(j0, min(j0 + width, n)) for j0 in range(0, n, width)]


def randomized_svd_blocked(a, k, p=10, q=0, seed=0, partitions=1):
    """rsvd_naive_ooc (rsvd.py:218-284): global power iteration where every
    product touching A is accumulated over column blocks with per-block
    slices of the sketch (gaussian_matrix row_offset, rsvd.py:236-245)."""
    m, n = a.shape
    l = k + p
    blocks = column_blocks(n, partitions)
    y = sum(a[:, j0:j1] @ normal_sketch(j1 - j0, l, seed, 0, j0, a.dtype)
            for j0, j1 in blocks)
    for _ in range(q):
        t = np.empty((n, l), dtype=a.dtype, order="F")
        for j0, j1 in blocks:
            t[j0:j1] = a[:, j0:j1].T @ y
        y = sum(a[:, j0:j1] @ t[j0:j1] for j0, j1 in blocks)
    qy, _, rank_y = orthonormal_range(y)
    b = np.empty((l, n), dtype=a.dtype, order="F")
    for j0, j1 in blocks:
        b[:, j0:j1] = qy.T @ a[:, j0:j1]
    w, s, vt, rank_b = core_svd(b)
    u, vt = canonical_signs(qy @ w, vt)
    return dict(U=u, sigma=s, Vt=vt, rank_y=rank_y, rank_b=rank_b)


def randomized_svd_paper(a, k, p, q, blocks, seed=0, omega=None):
    """brsvd_run with s > 1 (rsvd.py:150-215): the per-block power iteration
    of block_range_finder -- Y = sum_J (A_J A_J^T)^q A_J Omega_J with
    Omega_J = gaussian_matrix(|J|, l, seed, 0, row_offset=j0) (rsvd.py:169-175),
    no normalisation -- then Q = tsqr(Y), B[:, J] = Q^T A_J (rsvd.py:202-208)
    and _finish (rsvd.py:117-123)."""
    m, n = a.shape
    l = k + p
    y = None
    blocks = [(int(j0), int(j1)) for j0, j1 in blocks]   # Python ints: row << 192
    for j0, j1 in blocks:
        om = (omega[j0:j1] if omega is not None
              else normal_sketch(j1 - j0, l, seed, 0, j0, a.dtype))
        contrib = power_sample(a[:, j0:j1], om, q)
        y = contrib if y is None else y + contrib
    qy, _, rank_y = orthonormal_range(y)
    b = np.empty((l, n), dtype=a.dtype, order="F")
    for j0, j1 in blocks:
        b[:, j0:j1] = qy.T @ a[:, j0:j1]
    w, s, vt, rank_b = core_svd(b)
    u, vt = canonical_signs(qy @ w, vt)
    return dict(U=u, sigma=s, Vt=vt, rank_y=rank_y, rank_b=rank_b)


def range_basis_paper(a, k, p, q, blocks, seed=0, omega=None):
    """block_range_finder (rsvd.py:150-185): Q = tsqr of the per-block sample
    sum_J (A_J A_J^T)^q A_J Omega_J (rsvd.py:169-175, kernels.py:167-170)."""
    l = k + p
    y = None
    for j0, j1 in [(int(j0), int(j1)) for j0, j1 in blocks]:
        om = (omega[j0:j1] if omega is not None
              else normal_sketch(j1 - j0, l, seed, 0, j0, a.dtype))
        contrib = power_sample(a[:, j0:j1], om, q)
        y = contrib if y is None else y + contrib
    q_basis, _, rank = orthonormal_range(y)
    return q_basis, rank


def frob_rel_error(a, u, sigma, vt):
    """||A - U diag(s) Vt||_F / ||A||_F (rsvd.py:396-432, in-memory branch)."""
    d = a - (u * sigma) @ vt
    num, den = float(np.sum(d * d)), float(np.sum(a * a))
    if den == 0.0:
        return 0.0 if num == 0.0 else float("inf")
    return float(np.sqrt(num) / np.sqrt(den))


# --- rpca.py -------------------------------------------------------------------

def soft_threshold(x, eps):
    """sign(x) * max(|x| - eps, 0) (rpca.py:35-45)."""
    return np.sign(x) * np.maximum(np.abs(x) - eps, 0.0)


def power_norm(mat, seed=0, tol=1e-10, max_iterations=100):
    """Largest singular value by power iteration on M^T M (rpca.py:72-100):
    start from the stream-7 sketch column, stop when the estimate changes by
    at most tol relative."""
    v = normal_sketch(mat.shape[1], 1, seed, 7, dtype=mat.dtype)[:, 0]
    v = v / np.linalg.norm(v)
    est = 0.0
    for _ in range(max_iterations):
        u = mat @ v
        nu = np.linalg.norm(u)
        if nu == 0.0:
            return 0.0
        v = mat.T @ (u / nu)
        new = np.linalg.norm(v)
        v = v / new
        if abs(new - est) <= tol * new:
            return float(new)
        est = new
    return float(est)


def ialm(M, k, p=10, q=1, lam=None, mu0=None, rho=1.5, tol=1e-7,
         max_iterations=100, seed=0, blocks=None):
    """Inexact ALM robust PCA: in-core (rpca.py:168-213) or, with ``blocks``
    (the budget's column blocks), the out-of-core branch (rpca.py:216-304),
    whose inner SVD is brsvd_run's per-block power iteration (rpca.py:274).
    The out-of-core branch's block-wise W/L/S/Y updates are the same
    elementwise arithmetic as the in-core ones.

    Returns dict(L, S, iterations, residuals, mus, converged).
    """
    m, n = M.shape
    lam = 1.0 / np.sqrt(max(m, n)) if lam is None else lam
    norm2 = power_norm(M, seed=seed)
    if norm2 == 0.0:
        raise ValueError("RPCA input is the zero matrix")
    mu = 1.25 / norm2 if mu0 is None else mu0
    norm_f = np.linalg.norm(M)
    Y = M / max(norm2, np.max(np.abs(M)) / lam)
    S = np.zeros_like(M)
    L = None
    residuals, mus = [], []
    converged = False
    it = 0
    for it in range(1, max_iterations + 1):
        W = M - S + Y / mu
        f = (randomized_svd(W, k, p, q, seed) if blocks is None
             else randomized_svd_paper(W, k, p, q, blocks, seed=seed))
        L = (f["U"] * soft_threshold(f["sigma"], 1.0 / mu)) @ f["Vt"]
        S = soft_threshold(M - L + Y / mu, lam / mu)
        Z = M - L - S
        Y = Y + mu * Z
        r = float(np.linalg.norm(Z) / norm_f)
        residuals.append(r)
        mus.append(float(mu))
        if r < tol:
            converged = True
            break
        mu *= rho
    return dict(L=L, S=S, iterations=it, residuals=residuals, mus=mus,
                converged=converged)


# --- synthetic inputs (BASELINE.json configs) -----------------------------------

def lowrank_plus_noise(m, n, rank, noise, seed, dtype=np.float64):
    """A = L R + noise * N with iid N(0,1) factors."""
    rng = np.random.default_rng(seed)
    a = rng.standard_normal((m, rank)) @ rng.standard_normal((rank, n))
    if noise:
        a += noise * rng.standard_normal((m, n))
    return a.astype(dtype, copy=False)


def video_matrix(width, height, frames, seed=0, block=8, dtype=np.float64):
    """Synthetic surveillance video (BASELINE config 5 structure): each column
    is a width x height frame (column-major pixels), M = rank-3 nonnegative
    background + a block x block foreground square of value 1.0 that moves
    3 pixels per frame (wrapping), ~block^2 / (width*height) density."""
    rng = np.random.default_rng(seed)
    m = width * height
    M = rng.random((m, 3)) @ rng.random((3, frames))
    d = np.arange(block)
    y0 = height // 3
    for j in range(frames):
        x0 = (3 * j) % (width - block)
        rows = ((x0 + d)[:, None] * height + y0 + d[None, :]).ravel()
        M[rows, j] = 1.0
    return M.astype(dtype, copy=False)
