"""numpy stage operations for the row-sharded driver (TEST INFRASTRUCTURE).

Same interface as paper_1706_07191_b200.distributed.GpuOps, so the gloo tests
exercise the driver's sharding and collective logic on CPU; each operation
mirrors the semantics of the corresponding C ABI entry point.
"""

import numpy as np

from oracle import ref_cpu

F64 = np.float64


class NumpyOps:
    def dtype_of(self, A):
        return A.dtype

    def asarray(self, x, dtype):
        return np.asfortranarray(np.asarray(x), dtype=dtype)

    def absmax(self, A):
        return None   # scales of the fp16-split tensor-core products: GPU only

    def product(self, A, X, trans, amax=None):
        return np.asfortranarray((A.T if trans else A) @ X)

    def gram(self, X, W=None):
        W = X if W is None else W
        return np.asfortranarray(X.astype(F64).T @ W.astype(F64))

    def chol_basis(self, G, shift=0.0, col_drop=0.0, rank_tol=0.0, drop_ratio=0.0):
        """brsvd_chol_basis: scaled, column-order rank-revealing Cholesky."""
        G = np.array(G, dtype=F64)
        l = G.shape[0]
        d = np.diag(G).copy()
        dmax = d.max() if l else 0.0
        s = np.where((d > col_drop * col_drop * dmax) & (d > 0), 1.0 / np.sqrt(np.maximum(d, 1e-300)), 0.0)
        Gs = s[:, None] * (0.5 * (G + G.T)) * s[None, :] + shift * np.eye(l)
        diag0 = np.diag(Gs).copy()
        L = np.zeros((l, l))
        kept = []
        for j in range(l):
            piv = Gs[j, j] - L[j, :j] @ L[j, :j]
            ratio = piv / diag0[j] if diag0[j] > 0 and piv == piv else -1.0
            if (drop_ratio > 0 and not ratio > drop_ratio) or not piv > 0:
                L[j, j] = 1.0
                continue
            dj = np.sqrt(piv)
            L[j, j] = dj
            L[j + 1:, j] = (Gs[j + 1:, j] - L[j + 1:, :j] @ L[j, :j]) / dj
            kept.append(j)
        T = s[:, None] * np.linalg.inv(L).T
        out = np.zeros((l, l))
        out[:, :len(kept)] = T[:, kept]
        colnorm = np.where(s > 0, 1.0 / np.where(s > 0, s, 1.0), 0.0)
        cut = rank_tol * np.sqrt(np.sum(colnorm ** 2))
        rank = sum(1 for j in kept if s[j] > 0 and L[j, j] * colnorm[j] > cut) if rank_tol > 0 else 0
        return np.asfortranarray(out), len(kept), rank

    def apply(self, X, T, out_dtype, out=None, alpha=1.0, beta=0.0):
        r = alpha * (X.astype(F64) @ np.asarray(T, dtype=F64))
        if out is not None:
            if beta != 0.0:
                r = r + beta * out.astype(F64)
            out[...] = r.astype(out.dtype)
            return out
        return np.asfortranarray(r.astype(out_dtype))

    def normalize(self, Z):
        return self.normalize_t(Z, None)

    def normalize_t(self, Z, T_out):
        """brsvd_normalize_t: Zout = Z T, T kept (fp32 data: T rounded to fp32
        as the tensor-core basis change applies it)."""
        l = Z.shape[1]
        # unit scale first (exact power of two, folded into T), as
        # normalize_sketch does for fp64 operands near the exponent limits
        peak = float(np.max(np.abs(Z))) if Z.size else 0.0
        u = 2.0 ** -int(np.frexp(peak)[1]) if peak > 0 and np.isfinite(peak) else 1.0
        T, _, _ = self.chol_basis(self.gram(Z * u), shift=16.0 * l * 2.220446049250313e-16)
        T = T * u
        if Z.dtype == np.float32:
            T = T.astype(np.float32).astype(F64)
        if T_out is not None:
            T_out[...] = T
        return self.apply(Z, T, Z.dtype)

    def transform_buffers(self, q, l):
        return np.zeros((q, l, l))

    def unnormalised_peak(self, Y, Ts, zfac):
        """brsvd_unnormalised_peak: max |Y (prod zfac_i T_i)^-1| in fp64."""
        P = np.eye(Y.shape[1])
        scale = 1.0
        for T, z in zip(Ts, zfac):
            P = np.linalg.solve(np.asarray(T), P)
            scale *= z
        return float(np.max(np.abs(Y.astype(F64) @ P))) / scale if Y.size else 0.0

    def gaussian(self, rows, cols, seed, stream, row_offset, dtype):
        return ref_cpu.normal_sketch(int(rows), int(cols), seed % (2 ** 63), stream % (2 ** 63),
                                     int(row_offset), dtype)

    def small_svd(self, Bt):
        w, s, vt, rank = ref_cpu.core_svd(np.ascontiguousarray(Bt.T))
        return w.astype(F64), s, np.ascontiguousarray(vt), rank

    def colmax(self, U, row_offset):
        idx = np.argmax(np.abs(U), axis=0)
        vals = np.abs(U[idx, np.arange(U.shape[1])]).astype(F64)
        return vals, idx.astype(np.int64) + row_offset

    def entry(self, U, i, j):
        return float(U[i, j])

    def colmax_entries(self, U, row_offset):
        """brsvd_colmax_entries: [max |u| | global row | signed u] per column
        (NaN counts as +inf, like the kernel)."""
        a = np.abs(U).astype(F64)
        a[np.isnan(a)] = np.inf
        idx = np.argmax(a, axis=0)
        cols = np.arange(U.shape[1])
        return np.stack([a[idx, cols], (idx + row_offset).astype(F64),
                         U[idx, cols].astype(F64)])

    def stream_pass(self, shard, X, Y=None, want_z=False):
        """brsvd_stream_rows_pass: row panels of the host shard; Y_i = A_i X,
        Z += A_i^T Y_i summed in fp64."""
        a = shard.a
        m, n = a.shape
        if X is not None:
            Y = np.empty((m, X.shape[1]), dtype=a.dtype, order="F")
        Z = np.zeros((n, Y.shape[1]), dtype=F64, order="F") if want_z else None
        for r0 in range(0, m, shard.panel):
            r1 = min(m, r0 + shard.panel)
            if X is not None:
                Y[r0:r1] = a[r0:r1] @ X
            if want_z:
                Z += (a[r0:r1].T @ Y[r0:r1]).astype(F64)
        shard.passes += 1
        shard.pass_ms.append(0.0)
        return Y, Z

    def normalize_f64(self, Z, dtype, T=None):
        """brsvd_normalize_f64: fp32 data first at a power-of-two unit scale;
        with T also returns that scale (Zout = (s Z) T)."""
        s = 1.0
        if np.dtype(dtype) == np.float32:
            peak = float(np.max(np.abs(Z))) if Z.size else 0.0
            e = np.frexp(peak)[1] if peak > 0 else 0
            s = 2.0 ** -int(e)
            Z = np.asfortranarray((Z * s).astype(np.float32))
        out = self.normalize_t(np.asfortranarray(Z, dtype=dtype), T)
        return out if T is None else (out, s)

    def scale_cols(self, X, scale):
        X *= np.asarray(scale, dtype=X.dtype)[None, :]
        return X

    def hstack(self, a, b):
        return np.asfortranarray(np.hstack([a, b]))

    def cols(self, X, k):
        return X[:, :k]

    def cast(self, X, dtype):
        return np.asfortranarray(X.astype(dtype))
