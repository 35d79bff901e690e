"""Generate tests/golden/*.npz by running the REFERENCE package itself.

    PYTHONPATH=/root/reference/pkg/src python oracle/make_golden.py

Runs only in the build container (where /root/reference exists).  The
fixtures pin both the CPU oracle (oracle/ref_cpu.py, tests/test_oracle_golden.py)
and the GPU path (tests/test_gpu_parity.py, on the B200 box where
/root/reference is absent).  Inputs are stored alongside outputs so nothing
depends on regenerating random streams.
"""

import os
import sys
import warnings

import numpy as np

REF = "/root/reference/pkg/src"
if REF not in sys.path:
    sys.path.insert(0, REF)

import blocksvd as ref  # noqa: E402  (the reference package)

OUT = os.path.join(os.path.dirname(os.path.abspath(__file__)), "..", "tests", "golden")


def lowrank(m, n, k, seed, noise=0.0, dtype=np.float64):
    rng = np.random.default_rng(seed)
    a = rng.standard_normal((m, k)) @ rng.standard_normal((k, n))
    if noise:
        a = a + noise * rng.standard_normal((m, n))
    return a.astype(dtype)


def rsvd_case(name, a, k, p, q, seed):
    cfg = ref.SketchConfig(target_rank=k, oversampling=p, power_exponent=q,
                           master_seed=seed)
    omega = ref.gaussian_matrix(a.shape[1], k + p, seed, stream_index=0, dtype=a.dtype)
    with warnings.catch_warnings(record=True) as rec:
        warnings.simplefilter("always")
        f = ref.rsvd_incore(a, cfg)
    ranks = [w.message.detected_rank for w in rec
             if isinstance(w.message, ref.RankDeficiencyWarning)]
    err = ref.relative_frobenius_error(a, f)
    np.savez_compressed(os.path.join(OUT, f"rsvd_{name}.npz"), a=a, omega=omega,
                        k=k, p=p, q=q, seed=seed, U=f.U, sigma=f.sigma, Vt=f.Vt,
                        relerr=err, warned_ranks=np.array(ranks, dtype=np.int64))
    print(f"rsvd_{name}: sigma[:3]={f.sigma[:3]} relerr={err:.3e} ranks={ranks}")


def naive_ooc_case():
    """rsvd_naive_ooc (rsvd.py:218-284), global power iteration over column
    blocks; the global sketch is stored too (the per-block slices
    gaussian_matrix(|J|, l, seed, 0, row_offset=j0) are its rows,
    kernels.py:98-118)."""
    import tempfile
    a = lowrank(150, 100, 5, 14, noise=1e-6)
    with tempfile.TemporaryDirectory() as d:
        st = ref.MatrixStore.from_array(os.path.join(d, "a.oocm"), a)
        cfg = ref.SketchConfig(target_rank=5, power_exponent=2, partitions=5,
                               master_seed=3)
        with warnings.catch_warnings():
            warnings.simplefilter("ignore")
            fn, stats = ref.rsvd_naive_ooc(st, cfg)
        st.close()
    omega = ref.gaussian_matrix(100, 15, 3, stream_index=0)
    np.savez_compressed(os.path.join(OUT, "naive_ooc.npz"), a=a, U=fn.U,
                        sigma=fn.sigma, Vt=fn.Vt, passes=float(stats.full_passes),
                        omega=omega, k=5, p=10, q=2, s=5, seed=3,
                        block_reads=stats.block_reads)


def range_finder_case():
    """block_range_finder (rsvd.py:150-185): Q of the per-block sample."""
    import tempfile
    a = lowrank(240, 180, 6, 17, noise=1e-3)
    out = {}
    for s, q in ((1, 1), (3, 2)):
        with tempfile.TemporaryDirectory() as d:
            st = ref.MatrixStore.from_array(os.path.join(d, "a.oocm"), a)
            cfg = ref.SketchConfig(target_rank=6, oversampling=6, power_exponent=q,
                                   partitions=s, master_seed=11)
            with warnings.catch_warnings():
                warnings.simplefilter("ignore")
                Q, plan = ref.block_range_finder(st, cfg)
            out[f"Q_s{s}_q{q}"] = Q
            out[f"blocks_s{s}_q{q}"] = np.array(list(plan), dtype=np.int64)
            out[f"block_reads_s{s}_q{q}"] = st.stats.block_reads
            st.close()
    omega = ref.gaussian_matrix(180, 12, 11, stream_index=0)
    np.savez_compressed(os.path.join(OUT, "range_finder.npz"), a=a, omega=omega, **out)
    print("range_finder", sorted(out))


def rpca_video_case():
    """BASELINE config 5 structure at 1/10 of its columns and 1/10 of its
    pixels: a 96 x 80 video of 2000 frames (7680 x 2000 fp64, rank-3
    background + moving 8 x 8 foreground), k = p = 10, q = 1, tol 1e-7, run
    by the reference's ialm_rpca (rpca.py:168-213).  M is regenerated from
    oracle/ref_cpu.video_matrix (numpy default_rng; pinned by its checksum
    here); L and S are stored as probes (L @ P, P2^T L, norms) and the exact
    support and values of S."""
    from oracle import ref_cpu
    M = ref_cpu.video_matrix(96, 80, 2000, seed=0)
    cfg = ref.RpcaConfig(target_rank=10, oversampling=10, power_exponent=1, tol=1e-7)
    with warnings.catch_warnings():
        warnings.simplefilter("ignore")
        res = ref.ialm_rpca(M, cfg)
    omega = ref.gaussian_matrix(M.shape[1], 20, 0, stream_index=0)
    rng = np.random.default_rng(99)
    P = rng.standard_normal((M.shape[1], 4))
    P2 = rng.standard_normal((M.shape[0], 4))
    L, S = res.L, res.S
    nz = np.flatnonzero(S.ravel(order="F"))
    np.savez_compressed(os.path.join(OUT, "rpca_video_slice.npz"),
                        width=96, height=80, frames=2000, seed=0, k=10, p=10, q=1,
                        tol=1e-7, M_sum=M.sum(), M_sq=float((M * M).sum()), omega=omega,
                        P=P, P2=P2, LP=L @ P, P2L=P2.T @ L,
                        L_fro=np.linalg.norm(L), S_fro=np.linalg.norm(S),
                        S_idx=nz.astype(np.int64), S_val=S.ravel(order="F")[nz],
                        iterations=res.iterations,
                        residuals=np.array(res.residual_history),
                        mus=np.array([h["mu"] for h in res.history]),
                        converged=res.converged)
    print("rpca video slice iterations", res.iterations, "S nnz", nz.size)


CASES = {"naive_ooc": naive_ooc_case, "range_finder": range_finder_case,
         "rpca_video": rpca_video_case}


def main():
    os.makedirs(OUT, exist_ok=True)
    # rsvd_incore cases (rsvd.py:126-141)
    rsvd_case("c1small_f64", lowrank(1000, 200, 20, 11, noise=1e-3), 20, 10, 2, 0)
    rsvd_case("lr4_q0", lowrank(150, 90, 4, 6, noise=0.01), 4, 6, 0, 42)
    rsvd_case("lr4_q1", lowrank(150, 90, 4, 6, noise=0.01), 4, 6, 1, 42)
    rsvd_case("lr4_q2", lowrank(150, 90, 4, 6, noise=0.01), 4, 6, 2, 42)
    rsvd_case("exact_rank8", lowrank(100, 60, 8, 2), 8, 4, 1, 0)
    rsvd_case("f32_rank48", lowrank(1024, 384, 48, 5, noise=1e-3, dtype=np.float32),
              48, 8, 2, 0)
    rsvd_case("wide_f64", lowrank(80, 300, 6, 9, noise=1e-4), 6, 4, 1, 3)
    # decaying spectrum: sigma_i = 2^-i, sensitive to the sketch
    rng = np.random.default_rng(21)
    u, _ = np.linalg.qr(rng.standard_normal((400, 60)))
    v, _ = np.linalg.qr(rng.standard_normal((300, 60)))
    rsvd_case("decay_f64", (u * 0.7 ** np.arange(60)) @ v.T, 10, 10, 1, 7)

    # gaussian_matrix (kernels.py:98-118)
    g = ref.gaussian_matrix(50, 7, 123, stream_index=4)
    g_off = ref.gaussian_matrix(20, 7, 123, stream_index=4, row_offset=30)
    g32 = ref.gaussian_matrix(40, 5, 9, dtype=np.float32)
    np.savez_compressed(os.path.join(OUT, "gaussian.npz"), g=g, g_off=g_off, g32=g32)

    # tsqr (kernels.py:139-164)
    y = np.random.default_rng(3).standard_normal((1000, 12))
    q, r = ref.tsqr_factor(y, block_rows=100)
    yr = np.random.default_rng(6).standard_normal((200, 2)) @ \
        np.random.default_rng(7).standard_normal((2, 5))
    with warnings.catch_warnings(record=True) as rec:
        warnings.simplefilter("always")
        qr_, rr_ = ref.tsqr_factor(yr)
    rank = [w.message.detected_rank for w in rec][0]
    np.savez_compressed(os.path.join(OUT, "tsqr.npz"), y=y, q=q, r=r, y_def=yr,
                        q_def=qr_, rank_def=rank)

    # small_svd (kernels.py:173-188)
    b = np.random.default_rng(9).standard_normal((8, 20))
    f = ref.small_svd(b)
    bd = np.random.default_rng(11).standard_normal((4, 2)) @ \
        np.random.default_rng(12).standard_normal((2, 12))
    with warnings.catch_warnings():
        warnings.simplefilter("ignore")
        fd = ref.small_svd(bd)
    np.savez_compressed(os.path.join(OUT, "small_svd.npz"), b=b, W=f.U, sigma=f.sigma,
                        Vt=f.Vt, b_def=bd, sigma_def=fd.sigma)

    import tempfile

    # paper-literal two-pass BRSVD: brsvd_run with s > 1, q >= 1 computes the
    # per-block power iteration (rsvd.py:150-215)
    for name, a, k, p, q, s in (
            ("paper_s4_q2", lowrank(300, 240, 12, 31, noise=1e-2), 12, 8, 2, 4),
            ("paper_s3_q1", lowrank(200, 150, 6, 32, noise=1e-3), 6, 6, 1, 3)):
        with tempfile.TemporaryDirectory() as d:
            st = ref.MatrixStore.from_array(os.path.join(d, "a.oocm"), a)
            cfg = ref.SketchConfig(target_rank=k, oversampling=p, power_exponent=q,
                                   partitions=s, master_seed=5)
            with warnings.catch_warnings():
                warnings.simplefilter("ignore")
                fb, stats = ref.brsvd_run(st, cfg)
            plan = ref.plan_blocks(a.shape[1], a.shape[0], k + p, 8, s=s)
            st.close()
        omega = ref.gaussian_matrix(a.shape[1], k + p, 5, stream_index=0)
        np.savez_compressed(os.path.join(OUT, f"brsvd_{name}.npz"), a=a, omega=omega,
                            k=k, p=p, q=q, s=s, seed=5,
                            blocks=np.array(list(plan), dtype=np.int64),
                            U=fb.U, sigma=fb.sigma, Vt=fb.Vt,
                            passes=float(stats.full_passes))
        print(f"brsvd_{name}: sigma[:3]={fb.sigma[:3]} passes={stats.full_passes}")

    # RPCA (rpca.py:168-213)
    rng = np.random.default_rng(0)
    L0 = rng.standard_normal((200, 5)) @ rng.standard_normal((5, 200))
    mask = rng.random((200, 200)) < 0.05
    S0 = np.zeros((200, 200))
    S0[mask] = rng.choice([-1.0, 1.0], size=int(mask.sum())) * np.max(np.abs(L0))
    M = L0 + S0
    with warnings.catch_warnings():
        warnings.simplefilter("ignore")
        res = ref.ialm_rpca(M, ref.RpcaConfig(target_rank=10, tol=1e-7))
        n2 = ref.spectral_norm_estimate(M)
    omega = ref.gaussian_matrix(200, 20, 0, stream_index=0)
    np.savez_compressed(os.path.join(OUT, "rpca_planted.npz"), M=M, L0=L0, mask=mask,
                        omega=omega,
                        L=res.L, S=res.S, iterations=res.iterations,
                        residuals=np.array(res.residual_history),
                        mus=np.array([h["mu"] for h in res.history]),
                        converged=res.converged, norm2=n2)
    print("rpca iterations", res.iterations, "norm2", n2)

    # RPCA out-of-core branch (rpca.py:216-304): store input, budget below the
    # payload -> the inner SVD is brsvd_run over the budget's column blocks
    budget = 192000
    with tempfile.TemporaryDirectory() as d:
        st = ref.MatrixStore.from_array(os.path.join(d, "m.oocm"), M)
        cfgo = ref.RpcaConfig(target_rank=10, tol=1e-7, memory_budget_bytes=budget)
        with warnings.catch_warnings():
            warnings.simplefilter("ignore")
            reso = ref.ialm_rpca(st, cfgo)
        Lo, So = reso.L.read_full(), reso.S.read_full()
        plan = ref.plan_blocks(200, 200, 20, 8, memory_budget_bytes=budget)
        st.close()
    np.savez_compressed(os.path.join(OUT, "rpca_ooc.npz"), M=M, omega=omega, budget=budget,
                        blocks=np.array(list(plan), dtype=np.int64), L=Lo, S=So,
                        iterations=reso.iterations,
                        residuals=np.array(reso.residual_history),
                        converged=reso.converged)
    print("rpca ooc iterations", reso.iterations, "blocks", len(list(plan)))


if __name__ == "__main__":
    sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__)), ".."))
    if len(sys.argv) > 1:       # e.g. make_golden.py rpca_video naive_ooc
        for name in sys.argv[1:]:
            CASES[name]()
    else:
        main()
        for fn in CASES.values():
            fn()
