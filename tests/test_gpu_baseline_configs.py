"""Parity at the BASELINE.json configurations, against the CPU oracle or the
reference's own golden output (north-star tolerances):

  * config 2 at FULL size -- bench.make_matrix's 32768 x 32768 fp32
    rank-256 + 1e-3 noise, k=256 p=32 q=2 -- with the reference's sketch
    (ref_cpu.normal_sketch(32768, 288, 0, f32) == gaussian_matrix, pinned by
    test_oracle_golden.py) injected, against ref_cpu.randomized_svd run on the
    same host matrix (rsvd.py:126-141);
  * config 5's structure at 1/10 of its pixels and columns (a 96 x 80 x 2000
    video, fp64, k=p=10, q=1, tol 1e-7) against the reference's ialm_rpca
    output (tests/golden/rpca_video_slice.npz, rpca.py:168-213);
  * config 3's path -- a 2 GB row-major host matrix (5120 x 100000 fp32,
    rank-100 + noise, k=100 p=20 q=1) streamed through the panel streamer in
    row panels -- against ref_cpu.randomized_svd (rsvd.py:218-284 semantics).

Tolerances (BASELINE.json north_star): top-k sigma within 1e-5 relative
(fp32) / 1e-10 (fp64); principal-angle sine of U_k and V_k <= 1e-4;
|relerr - relerr_ref| <= 1e-4; RPCA: same iteration count, L within 1e-6.
"""

import os
import warnings

import numpy as np
import pytest

from oracle import ref_cpu
from tests.conftest import GOLDEN

pytestmark = pytest.mark.gpu


def sin_theta(u, v):
    """Sine of the largest principal angle, fp64."""
    qu, _ = np.linalg.qr(np.asarray(u, dtype=np.float64))
    qv, _ = np.linalg.qr(np.asarray(v, dtype=np.float64))
    return float(np.linalg.norm(qu - qv @ (qv.T @ qu), 2))


def relerr_torch(A, U, s, Vt, chunk=4096):
    """||A - U diag(s) Vt||_F / ||A||_F in fp64 with torch on the device (an
    independent checker: cuBLAS fp64, not the product path)."""
    import torch
    dev = A.device
    U = torch.as_tensor(np.asarray(U), device=dev).double()
    Vs = (torch.as_tensor(np.asarray(Vt), device=dev).double()
          * torch.as_tensor(np.asarray(s), device=dev).double()[:, None])
    num = den = 0.0
    for r0 in range(0, A.shape[0], chunk):
        a = A[r0:r0 + chunk].double()
        d = a - U[r0:r0 + chunk] @ Vs
        num += float((d * d).sum())
        den += float((a * a).sum())
    return (num / den) ** 0.5


@pytest.fixture(autouse=True)
def quiet():
    from paper_1706_07191_b200 import RankDeficiencyWarning
    with warnings.catch_warnings():
        warnings.simplefilter("ignore", RankDeficiencyWarning)
        warnings.simplefilter("ignore", RuntimeWarning)   # the reference's fp32 norm overflows
        yield


def test_config2_full_size_matches_oracle():
    import torch
    import bench
    from paper_1706_07191_b200 import SketchConfig, rsvd_incore
    A = bench.make_matrix(torch.device("cuda:0"))
    a = A.cpu().numpy()
    k, p, q = bench.K, bench.P, bench.Q
    omega = ref_cpu.normal_sketch(a.shape[1], k + p, 0, dtype=np.float32)
    ref = ref_cpu.randomized_svd(a, k, p, q, seed=0, omega=omega)
    f = rsvd_incore(A, SketchConfig(k, p, q, master_seed=0), omega=omega)
    sig = f.sigma.cpu().numpy()
    U, Vt = f.U.cpu().numpy(), f.Vt.cpu().numpy()
    rel = np.max(np.abs(sig[:k].astype(np.float64) - ref["sigma"][:k]) / ref["sigma"][:k])
    assert rel <= 1e-5, rel
    assert sin_theta(U[:, :k], ref["U"][:, :k]) <= 1e-4
    assert sin_theta(Vt[:k].T, ref["Vt"][:k].T) <= 1e-4
    e_gpu = relerr_torch(A, U[:, :k], sig[:k], Vt[:k])
    e_ref = relerr_torch(A, ref["U"][:, :k], ref["sigma"][:k], ref["Vt"][:k])
    assert abs(e_gpu - e_ref) <= 1e-4, (e_gpu, e_ref)
    # canonical signs (rsvd.py:105-115): the leading vectors agree entrywise
    np.testing.assert_allclose(U[:, :8], ref["U"][:, :8], atol=1e-3)


def test_config5_slice_matches_reference_golden():
    from paper_1706_07191_b200 import RpcaConfig, ialm_rpca
    g = np.load(os.path.join(GOLDEN, "rpca_video_slice.npz"))
    M = ref_cpu.video_matrix(int(g["width"]), int(g["height"]), int(g["frames"]),
                             seed=int(g["seed"]))
    assert M.sum() == float(g["M_sum"])
    cfg = RpcaConfig(target_rank=int(g["k"]), oversampling=int(g["p"]),
                     power_exponent=int(g["q"]), tol=float(g["tol"]))
    res = ialm_rpca(M, cfg, omega=g["omega"])
    assert res.converged and res.iterations == int(g["iterations"])
    np.testing.assert_allclose([h["mu"] for h in res.history], g["mus"], rtol=1e-8)
    np.testing.assert_allclose(res.residual_history, g["residuals"], rtol=1e-4)
    L, S = res.L, res.S
    for got, want in ((L @ g["P"], g["LP"]), (g["P2"].T @ L, g["P2L"])):
        assert np.linalg.norm(got - want) <= 1e-6 * np.linalg.norm(want)
    assert abs(np.linalg.norm(L) - float(g["L_fro"])) <= 1e-6 * float(g["L_fro"])
    s_flat = S.ravel(order="F")
    nz = np.flatnonzero(s_flat)
    ref_idx, ref_val = g["S_idx"], g["S_val"]
    # support: entries of the reference's S at the soft-threshold edge may flip
    sym = np.setxor1d(nz, ref_idx).size
    assert sym <= 1e-3 * ref_idx.size, (sym, ref_idx.size)
    dense_ref = np.zeros_like(s_flat)
    dense_ref[ref_idx] = ref_val
    assert np.linalg.norm(s_flat - dense_ref) <= 1e-6 * np.linalg.norm(ref_val)


def test_config3_path_2gb_stream_matches_oracle():
    import torch
    from paper_1706_07191_b200 import SketchConfig
    from paper_1706_07191_b200.rsvd import run_rsvd_stream
    m, n, rank, k, p, q = 5120, 100000, 100, 100, 20, 1
    g = torch.Generator(device="cuda").manual_seed(31)
    A = (torch.randn(m, rank, generator=g, device="cuda")
         @ torch.randn(rank, n, generator=g, device="cuda"))
    A.add_(torch.randn(m, n, generator=g, device="cuda"), alpha=1e-3)
    host = torch.empty((m, n), dtype=torch.float32, pin_memory=True)
    host.copy_(A)
    a = host.numpy()                                   # 2.05 GB, row-major, pinned
    omega = ref_cpu.normal_sketch(n, k + p, 0, dtype=np.float32)
    run = run_rsvd_stream(a, SketchConfig(k, p, q), panel=1024, nbuf=3, omega=omega,
                          warn=False)
    assert run.stats.words_read == (q + 2) * m * n
    ref = ref_cpu.randomized_svd(a, k, p, q, seed=0, omega=omega)
    f = run.factors
    rel = np.max(np.abs(f.sigma[:k].astype(np.float64) - ref["sigma"][:k]) / ref["sigma"][:k])
    assert rel <= 1e-5, rel
    assert sin_theta(f.U[:, :k], ref["U"][:, :k]) <= 1e-4
    assert sin_theta(f.Vt[:k].T, ref["Vt"][:k].T) <= 1e-4
    e_gpu = relerr_torch(A, f.U[:, :k], f.sigma[:k], f.Vt[:k])
    e_ref = relerr_torch(A, ref["U"][:, :k], ref["sigma"][:k], ref["Vt"][:k])
    assert abs(e_gpu - e_ref) <= 1e-4, (e_gpu, e_ref)
