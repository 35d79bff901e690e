"""GPU parity: the CUDA path (through the C ABI) against the reference.

Two anchors:
  * tests/golden/*.npz -- outputs of the reference package itself
    (oracle/make_golden.py), with the reference's own Omega injected so both
    sides see the same sketch;
  * oracle/ref_cpu.py run live on the same seeded inputs at BASELINE config 1
    (the CPU oracle is pinned to the golden vectors by test_oracle_golden.py).

Tolerances are the north star's (BASELINE.json): top-k singular values within
1e-10 relative (fp64) / 1e-5 (fp32); principal-angle sine and relative
reconstruction error within 1e-4 of the reference's values.
"""

import os
import warnings

import numpy as np
import pytest

from oracle import ref_cpu
from tests.conftest import GOLDEN

pytestmark = pytest.mark.gpu


def load(name):
    return np.load(os.path.join(GOLDEN, name))


def sin_theta(u, v):
    """sin of the largest principal angle between range(u) and range(v)
    (sine form), in fp64."""
    qu, _ = np.linalg.qr(np.asarray(u, dtype=np.float64))
    qv, _ = np.linalg.qr(np.asarray(v, dtype=np.float64))
    return float(np.linalg.norm(qu - qv @ (qv.T @ qu), 2))


@pytest.fixture(autouse=True)
def quiet():
    from paper_1706_07191_b200 import RankDeficiencyWarning
    with warnings.catch_warnings():
        warnings.simplefilter("ignore", RankDeficiencyWarning)
        yield


RSVD_CASES = ["c1small_f64", "lr4_q0", "lr4_q1", "lr4_q2", "exact_rank8", "f32_rank48",
              "wide_f64", "decay_f64"]


@pytest.mark.parametrize("case", RSVD_CASES)
def test_rsvd_matches_reference_golden(case):
    from paper_1706_07191_b200 import SketchConfig, rsvd_incore
    g = load(f"rsvd_{case}.npz")
    a = g["a"]
    k, p, q, seed = int(g["k"]), int(g["p"]), int(g["q"]), int(g["seed"])
    cfg = SketchConfig(target_rank=k, oversampling=p, power_exponent=q, master_seed=seed)
    f = rsvd_incore(a, cfg, omega=g["omega"])
    assert f.U.shape == (a.shape[0], k + p) and f.Vt.shape == (k + p, a.shape[1])
    assert f.U.dtype == a.dtype and f.sigma.dtype == a.dtype
    fp64 = a.dtype == np.float64
    rtol = 1e-10 if fp64 else 1e-5
    np.testing.assert_allclose(f.sigma[:k], g["sigma"][:k], rtol=rtol)
    assert np.all(np.diff(f.sigma.astype(np.float64)) <= 0)
    assert sin_theta(f.U[:, :k], g["U"][:, :k]) <= (1e-8 if fp64 else 1e-4)
    assert sin_theta(f.Vt[:k].T, g["Vt"][:k].T) <= (1e-8 if fp64 else 1e-4)
    err = ref_cpu.frob_rel_error(a.astype(np.float64), f.U.astype(np.float64),
                                 f.sigma.astype(np.float64), f.Vt.astype(np.float64))
    assert abs(err - float(g["relerr"])) <= 1e-4
    # canonical signs (rsvd.py:105-115): leading vectors agree entrywise
    atol = 1e-7 if fp64 else 2e-3
    np.testing.assert_allclose(f.U[:, :k], g["U"][:, :k], atol=atol)


def test_factor_contracts_rank_deficient():
    """tests/test_rsvd.py:62-71 of the reference, on the GPU."""
    from paper_1706_07191_b200 import SketchConfig, rsvd_incore
    g = load("rsvd_exact_rank8.npz")
    f = rsvd_incore(g["a"], SketchConfig(target_rank=8, oversampling=4, power_exponent=1),
                    omega=g["omega"])
    l, eps = 12, np.finfo(np.float64).eps
    assert f.effective_l == l
    assert np.linalg.norm(f.U.T @ f.U - np.eye(l)) <= 100 * l * eps
    assert np.linalg.norm(f.Vt @ f.Vt.T - np.eye(l)) <= 100 * l * eps
    assert np.all(np.diff(f.sigma) <= 0)


def test_rank_warnings_like_reference():
    from paper_1706_07191_b200 import RankDeficiencyWarning, SketchConfig, rsvd_incore
    g = load("rsvd_exact_rank8.npz")
    with warnings.catch_warnings(record=True) as rec:
        warnings.simplefilter("always")
        rsvd_incore(g["a"], SketchConfig(target_rank=8, oversampling=4, power_exponent=1))
    ranks = [w.message.detected_rank for w in rec
             if isinstance(w.message, RankDeficiencyWarning)]
    assert ranks == list(g["warned_ranks"])


def test_config1_full_size_against_live_oracle():
    """BASELINE config 1: 10000x2000 fp64 rank-20 + 1e-3 noise, k=20 p=10 q=2."""
    from paper_1706_07191_b200 import SketchConfig, rsvd_incore
    a = ref_cpu.lowrank_plus_noise(10000, 2000, 20, 1e-3, seed=1)
    ref = ref_cpu.randomized_svd(a, 20, 10, 2, seed=0)
    f = rsvd_incore(a, SketchConfig(20, 10, 2, master_seed=0), omega=ref["omega"])
    np.testing.assert_allclose(f.sigma[:20], ref["sigma"][:20], rtol=1e-10)
    assert sin_theta(f.U[:, :20], ref["U"][:, :20]) <= 1e-8
    e_gpu = ref_cpu.frob_rel_error(a, f.U, f.sigma, f.Vt)
    e_ref = ref_cpu.frob_rel_error(a, ref["U"], ref["sigma"], ref["Vt"])
    assert abs(e_gpu - e_ref) <= 1e-4


def test_column_major_and_device_inputs_agree():
    import torch
    from paper_1706_07191_b200 import SketchConfig, rsvd_incore
    g = load("rsvd_lr4_q2.npz")
    a, om = g["a"], g["omega"]
    cfg = SketchConfig(4, 6, 2, master_seed=42)
    f_c = rsvd_incore(np.ascontiguousarray(a), cfg, omega=om)
    f_f = rsvd_incore(np.asfortranarray(a), cfg, omega=om)
    f_d = rsvd_incore(torch.as_tensor(a, device="cuda"), cfg, omega=om)
    for f in (f_f,):
        np.testing.assert_allclose(f.sigma, f_c.sigma, rtol=1e-12)
    np.testing.assert_allclose(f_d.sigma.cpu().numpy(), f_c.sigma, rtol=1e-12)
    np.testing.assert_allclose(f_d.U.cpu().numpy()[:, :4], f_c.U[:, :4], atol=1e-10)


def test_deterministic_for_seed():
    """tests/test_rsvd.py:79-82: identical inputs give bit-identical factors."""
    from paper_1706_07191_b200 import SketchConfig, rsvd_incore
    a = np.asfortranarray(ref_cpu.lowrank_plus_noise(80, 50, 6, 0.0, seed=4))
    cfg = SketchConfig(target_rank=6, master_seed=9)
    f1, f2 = rsvd_incore(a, cfg), rsvd_incore(a, cfg)
    assert np.array_equal(f1.U, f2.U) and np.array_equal(f1.sigma, f2.sigma)
    assert np.array_equal(f1.Vt, f2.Vt)


def test_generated_sketch_gives_reference_quality():
    """Without injection the GPU sketch differs from numpy's stream, but the
    captured spectrum is the same (tests/test_rsvd.py:44-53)."""
    from paper_1706_07191_b200 import SketchConfig, rsvd_incore
    rng = np.random.default_rng(1)
    u, _ = np.linalg.qr(rng.standard_normal((50, 50)))
    v, _ = np.linalg.qr(rng.standard_normal((40, 40)))
    s = np.concatenate([np.linspace(10.0, 1.0, 10), np.full(30, 1e-3)])
    a = u[:, :40] @ (s[:, None] * v.T)
    f = rsvd_incore(a, SketchConfig(target_rank=10, power_exponent=2))
    dense = np.linalg.svd(a, compute_uv=False)
    np.testing.assert_allclose(f.sigma[:10], dense[:10], rtol=1e-8)


def test_exact_rank4_reconstruction_and_diagonal():
    from paper_1706_07191_b200 import SketchConfig, relative_frobenius_error, rsvd_incore
    rng = np.random.default_rng(0)
    a = rng.standard_normal((1024, 4)) @ rng.standard_normal((4, 64))
    f = rsvd_incore(a, SketchConfig(target_rank=4, oversampling=10, power_exponent=1))
    assert relative_frobenius_error(a, f) <= 1e-12
    d = np.diag([5.0, 4.0, 3.0, 2.0, 1.0])
    f = rsvd_incore(d, SketchConfig(target_rank=5, oversampling=0, power_exponent=0))
    np.testing.assert_allclose(f.sigma, [5, 4, 3, 2, 1], atol=1e-12)


def test_overflow_guard_raises():
    """tests/test_rsvd.py:162-169: unnormalised power iteration would overflow."""
    from paper_1706_07191_b200 import SketchConfig, rsvd_incore
    rng = np.random.default_rng(11)
    a = 1e30 * (rng.standard_normal((40, 2)) @ rng.standard_normal((2, 30)))
    with pytest.raises(FloatingPointError):
        rsvd_incore(a, SketchConfig(target_rank=2, power_exponent=10, q_max=10))
    with pytest.raises(FloatingPointError):
        bad = np.ones((20, 10))
        bad[3, 4] = np.inf
        rsvd_incore(bad, SketchConfig(target_rank=2, oversampling=2))


def test_config_errors_before_device_work():
    from paper_1706_07191_b200 import ConfigError, SketchConfig, rsvd_incore
    with pytest.raises(ConfigError):
        rsvd_incore(np.ones((10, 8)), SketchConfig(target_rank=5, oversampling=5))


def test_tsqr_against_golden():
    from paper_1706_07191_b200 import RankDeficiencyWarning, tsqr, tsqr_factor
    g = load("tsqr.npz")
    y = g["y"]
    q, r = tsqr_factor(y, block_rows=100)
    l, eps = y.shape[1], np.finfo(np.float64).eps
    assert np.linalg.norm(q.T @ q - np.eye(l)) <= 100 * l * eps
    np.testing.assert_allclose(q @ r, y, atol=1e-12 * np.abs(y).max())
    proj = q @ q.T - g["q"] @ g["q"].T
    assert np.linalg.norm(proj) <= 1e-12
    # full rank: R upper triangular, as the reference's Householder R
    assert np.all(np.tril(r, -1) == 0.0)
    with pytest.warns(RankDeficiencyWarning) as rec:
        qd, _ = tsqr_factor(g["y_def"])
    assert rec[0].message.detected_rank == int(g["rank_def"])
    assert np.allclose(qd.T @ qd, np.eye(5), atol=1e-12)
    e = np.zeros((4, 2))
    e[0, 0] = e[1, 1] = 1.0
    assert np.allclose(np.abs(tsqr(e)), e)


def test_small_svd_against_golden():
    from paper_1706_07191_b200 import RankDeficiencyWarning, small_svd
    g = load("small_svd.npz")
    f = small_svd(g["b"])
    np.testing.assert_allclose(f.sigma, g["sigma"], rtol=1e-10)
    np.testing.assert_allclose(np.abs(f.U), np.abs(g["W"]), atol=1e-10)
    err = np.linalg.norm(g["b"] - f.compose()) / np.linalg.norm(g["b"])
    assert err <= 6 * 100 * np.finfo(np.float64).eps
    with pytest.warns(RankDeficiencyWarning):
        fd = small_svd(g["b_def"])
    assert fd.sigma[2] <= 1e-12 * fd.sigma[0] and fd.sigma[3] <= 1e-12 * fd.sigma[0]
    np.testing.assert_allclose(fd.sigma[:2], g["sigma_def"][:2], rtol=1e-10)


def test_gaussian_matrix_properties():
    """tests/test_kernels.py:61-89 properties of the device generator."""
    from paper_1706_07191_b200 import ShapeError, gaussian_matrix
    g1 = gaussian_matrix(50, 7, 123, stream_index=4)
    assert np.array_equal(g1, gaussian_matrix(50, 7, 123, stream_index=4))
    full = gaussian_matrix(200, 5, 11)
    assert np.array_equal(full[140:], gaussian_matrix(60, 5, 11, row_offset=140))
    g = gaussian_matrix(10000, 100, 99)
    assert abs(g.mean()) <= 0.01 and abs(g.var() - 1.0) <= 0.01
    a = gaussian_matrix(10000, 10, 5, stream_index=0).ravel()
    b = gaussian_matrix(10000, 10, 5, stream_index=1).ravel()
    assert abs(np.corrcoef(a, b)[0, 1]) <= 0.01
    assert gaussian_matrix(100, 4, 0, dtype=np.float32).dtype == np.float32
    with pytest.raises(ShapeError):
        gaussian_matrix(0, 3, 1)


def test_f32_config2_shape_small_scale():
    """Config 2 structure (square fp32, rank-256+noise, k=256 p=32 q=2) at 4096^2."""
    from paper_1706_07191_b200 import SketchConfig, rsvd_incore
    a = ref_cpu.lowrank_plus_noise(4096, 4096, 256, 1e-3, seed=2, dtype=np.float32)
    omega = ref_cpu.normal_sketch(4096, 288, 0, dtype=np.float32)
    ref = ref_cpu.randomized_svd(a, 256, 32, 2, seed=0, omega=omega)
    f = rsvd_incore(a, SketchConfig(256, 32, 2), omega=omega)
    np.testing.assert_allclose(f.sigma[:256], ref["sigma"][:256], rtol=1e-5)
    assert sin_theta(f.U[:, :256], ref["U"][:, :256]) <= 1e-3
    a64 = a.astype(np.float64)
    e_gpu = ref_cpu.frob_rel_error(a64, f.U.astype(np.float64), f.sigma.astype(np.float64),
                                   f.Vt.astype(np.float64))
    e_ref = ref_cpu.frob_rel_error(a64, ref["U"].astype(np.float64),
                                   ref["sigma"].astype(np.float64),
                                   ref["Vt"].astype(np.float64))
    assert abs(e_gpu - e_ref) <= 1e-4


@pytest.mark.parametrize("order", ["C", "F"])
@pytest.mark.parametrize("dtype", [np.float64, np.float32])
def test_streamed_out_of_core_matches_in_core(order, dtype):
    """brsvd_rsvd_stream (host-resident A, panels over PCIe) == in-core."""
    from paper_1706_07191_b200 import SketchConfig
    from paper_1706_07191_b200.rsvd import run_rsvd, run_rsvd_stream
    a = ref_cpu.lowrank_plus_noise(3000, 1200, 20, 1e-3, seed=21, dtype=dtype)
    a = np.asarray(a, order=order)
    omega = ref_cpu.normal_sketch(1200, 30, 0, dtype=dtype)
    cfg = SketchConfig(20, 10, 2)
    inc = run_rsvd(a, cfg, omega=omega, warn=False)
    st = run_rsvd_stream(a, cfg, panel=257, nbuf=3, omega=omega, warn=False)
    assert st.stats.words_read == (2 + 2) * a.size          # q + 2 passes
    fp64 = dtype == np.float64
    np.testing.assert_allclose(st.factors.sigma[:20], inc.factors.sigma[:20],
                               rtol=1e-10 if fp64 else 1e-5)
    assert sin_theta(st.factors.U[:, :20], inc.factors.U[:, :20]) <= (1e-8 if fp64 else 1e-4)
    ref = ref_cpu.randomized_svd(a, 20, 10, 2, omega=omega)
    np.testing.assert_allclose(st.factors.sigma[:20], ref["sigma"][:20],
                               rtol=1e-10 if fp64 else 1e-5)


def test_brsvd_run_budget_streams_store(tmp_path):
    """brsvd_run with a budget below the payload streams the plan's blocks;
    PassStats keeps the reference's accounting (rsvd.py:188-193: two passes,
    2 s block reads) and boundary_words_read the true PCIe traffic."""
    from paper_1706_07191_b200 import MatrixStore, SketchConfig, brsvd_run, rsvd_incore
    a = ref_cpu.lowrank_plus_noise(2000, 600, 8, 1e-4, seed=22)
    st = MatrixStore.from_array(tmp_path / "a.oocm", a)
    cfg = SketchConfig(target_rank=8, oversampling=8, power_exponent=1)
    f, stats = brsvd_run(st, cfg, memory_budget_bytes=4 * 1024 * 1024, mode="global")
    assert stats.full_passes == 2 and stats.words_read == 2 * a.size
    assert stats.boundary_words_read == 3 * a.size              # q + 2 streamed passes
    assert [e["stage"] for e in stats.stage_log] == ["sketch", "orthonormalize",
                                                     "form_core", "svd"]
    g = rsvd_incore(a, cfg)
    np.testing.assert_allclose(f.sigma[:8], g.sigma[:8], rtol=1e-10)
    f2, stats2 = brsvd_run(st, cfg, mode="global")             # fits: landed once
    assert stats2.full_passes == 2 and stats2.block_reads == 2
    assert stats2.boundary_words_read == a.size
    np.testing.assert_allclose(f2.sigma[:8], g.sigma[:8], rtol=1e-10)
    st.close()


@pytest.mark.parametrize("name", ["brsvd_paper_s4_q2.npz", "brsvd_paper_s3_q1.npz"])
def test_brsvd_run_matches_reference_through_public_api(name, tmp_path):
    """brsvd_run (default: the reference's per-block power iteration,
    rsvd.py:150-215) with the reference's Omega injected reproduces the
    reference's factors, in HBM and streamed in the plan's column blocks, with
    the reference's pass law (full_passes == 2, block_reads == 2 s)."""
    from paper_1706_07191_b200 import MatrixStore, SketchConfig, brsvd_run
    g = load(name)
    a = g["a"]
    k, p, q, s = int(g["k"]), int(g["p"]), int(g["q"]), int(g["s"])
    st = MatrixStore.from_array(tmp_path / "a.oocm", a)
    cfg = SketchConfig(target_rank=k, oversampling=p, power_exponent=q, partitions=s,
                       master_seed=int(g["seed"]))
    budget = 3 * a.shape[0] * (k + p) * 8 + 10 * a.shape[0] * 8
    for bud in (None, budget):
        f, stats = brsvd_run(st, cfg, memory_budget_bytes=bud, omega=g["omega"])
        assert stats.full_passes == 2
        if bud is None:
            assert stats.block_reads == 2 * len(g["blocks"])
        np.testing.assert_allclose(f.sigma[:k], g["sigma"][:k], rtol=1e-10)
        assert sin_theta(f.U[:, :k], g["U"][:, :k]) <= 1e-8
        assert sin_theta(f.Vt[:k].T, g["Vt"][:k].T) <= 1e-8
        np.testing.assert_allclose(f.U[:, :k], g["U"][:, :k], atol=1e-8)
    assert stats.boundary_words_read == 2 * a.size           # streamed: 2 passes
    # the per-block sample is a different approximation from the global one
    glob, _ = brsvd_run(st, cfg, mode="global", omega=g["omega"])
    gap = np.max(np.abs(glob.sigma[:k] - f.sigma[:k]) / f.sigma[:k])
    assert gap > (1e-6 if "s4_q2" in name else 0.0)
    st.close()


def test_naive_ooc_matches_reference_golden(tmp_path):
    """rsvd_naive_ooc (rsvd.py:218-284) with the reference's sketch: global
    power iteration, factors to 1e-10, pass law 2(q + 1) (test_rsvd.py:173-179)."""
    from paper_1706_07191_b200 import MatrixStore, SketchConfig, rsvd_naive_ooc
    g = load("naive_ooc.npz")
    a = g["a"]
    k, p, q, s = int(g["k"]), int(g["p"]), int(g["q"]), int(g["s"])
    st = MatrixStore.from_array(tmp_path / "a.oocm", a)
    cfg = SketchConfig(target_rank=k, oversampling=p, power_exponent=q, partitions=s,
                       master_seed=int(g["seed"]))
    f, stats = rsvd_naive_ooc(st, cfg, omega=g["omega"])
    st.close()
    assert stats.full_passes == float(g["passes"]) == 2 * (q + 1)
    assert stats.block_reads == int(g["block_reads"])
    assert [e["stage"] for e in stats.stage_log] == ["sketch", "power", "orthonormalize",
                                                     "form_core", "svd"]
    np.testing.assert_allclose(f.sigma[:k], g["sigma"][:k], rtol=1e-10)
    assert sin_theta(f.U[:, :k], g["U"][:, :k]) <= 1e-8
    np.testing.assert_allclose(f.U[:, :k], g["U"][:, :k], atol=1e-8)


@pytest.mark.parametrize("s,q", [(1, 1), (3, 2)])
def test_block_range_finder_matches_reference(s, q, tmp_path):
    """block_range_finder (rsvd.py:150-185): the orthonormal basis of the
    per-block sample, no core projection; one pass added to the store's
    counters (not reset)."""
    from paper_1706_07191_b200 import MatrixStore, SketchConfig, block_range_finder
    g = load("range_finder.npz")
    a = g["a"]
    st = MatrixStore.from_array(tmp_path / "a.oocm", a)
    cfg = SketchConfig(target_rank=6, oversampling=6, power_exponent=q, partitions=s,
                       master_seed=11)
    Q, plan = block_range_finder(st, cfg, omega=g["omega"])
    assert [tuple(b) for b in plan] == [tuple(b) for b in g[f"blocks_s{s}_q{q}"]]
    assert st.stats.block_reads == int(g[f"block_reads_s{s}_q{q}"]) == s
    assert st.stats.full_passes == 1
    Qr = g[f"Q_s{s}_q{q}"]
    assert Q.shape == Qr.shape and np.linalg.norm(Q.T @ Q - np.eye(12)) <= 1e-12
    # the leading columns span the same nested subspaces as the reference's
    # Householder Q (both orthonormalise in column order) ...
    assert np.linalg.norm(Q[:, :6] @ Q[:, :6].T - Qr[:, :6] @ Qr[:, :6].T) <= 1e-10
    # ... and Q captures the reference's sample (range residual as in the
    # reference's tests/test_kernels.py:100-108)
    y = None
    for j0, j1 in plan:
        c = ref_cpu.power_sample(a[:, j0:j1], g["omega"][j0:j1], q)
        y = c if y is None else y + c
    assert np.linalg.norm(y - Q @ (Q.T @ y)) <= 1e-12 * np.linalg.norm(y)
    block_range_finder(st, cfg, omega=g["omega"])
    assert st.stats.full_passes == 2                        # accumulates like the reference
    st.close()


def test_paper_mode_with_reference_omega_is_bit_close():
    """Same A, same Omega (the reference's), same blocks: the per-block sketch
    through the C ABI (brsvd_rsvd_blocked) reproduces the reference's
    brsvd_run factors to rounding."""
    from paper_1706_07191_b200 import SketchConfig
    from paper_1706_07191_b200.rsvd import run_rsvd
    for name in ("brsvd_paper_s4_q2.npz", "brsvd_paper_s3_q1.npz"):
        g = load(name)
        a = np.asfortranarray(g["a"])
        k, p, q = int(g["k"]), int(g["p"]), int(g["q"])
        blocks = [(int(j0), int(j1)) for j0, j1 in g["blocks"]]
        cfg = SketchConfig(target_rank=k, oversampling=p, power_exponent=q)
        with warnings.catch_warnings():
            warnings.simplefilter("ignore")
            f = run_rsvd(a, cfg, omega=g["omega"], blocks=blocks).factors
        np.testing.assert_allclose(f.sigma[:k], g["sigma"][:k], rtol=1e-10)
        s_ang = sin_theta(f.U[:, :k], g["U"][:, :k])
        assert s_ang <= 1e-8


@pytest.mark.parametrize("scale,q", [(1e-30, 2), (1e-20, 1), (1e-12, 2), (1e12, 0),
                                     (1e30, 0)])
def test_f32_scale_invariance(scale, q):
    """fp32 inputs far from unit magnitude: the fp16-split product rescales
    rows/columns by powers of two, A^T Y of the power iteration is taken at a
    power-of-two scale, and the Grams/Cholesky/Jacobi run in fp64, so the
    factorization of s*A is s times that of A (to fp32 accuracy).  (Large s
    with q > 0 trips the reference's overflow guard by design.)"""
    from paper_1706_07191_b200 import SketchConfig, rsvd_incore
    a = ref_cpu.lowrank_plus_noise(2048, 1536, 64, 1e-3, seed=4, dtype=np.float32)
    omega = ref_cpu.normal_sketch(1536, 80, 0, dtype=np.float32)
    f1 = rsvd_incore(a, SketchConfig(64, 16, q), omega=omega)
    As = (a.astype(np.float64) * scale).astype(np.float32)
    import torch
    for inp in (As, torch.from_numpy(As).cuda()):      # host feed and device paths
        fs = rsvd_incore(inp, SketchConfig(64, 16, q), omega=omega)
        sig = np.asarray(fs.sigma.cpu() if hasattr(fs.sigma, "cpu") else fs.sigma)
        np.testing.assert_allclose(sig[:64] / scale, f1.sigma[:64], rtol=1e-5)
        U = np.asarray(fs.U.cpu() if hasattr(fs.U, "cpu") else fs.U)
        assert sin_theta(U[:, :64], f1.U[:, :64]) <= 1e-3


@pytest.mark.parametrize("order", ["C", "F"])
@pytest.mark.parametrize("scale", [1e-30, 1e-20])
def test_streamed_scale_invariance(order, scale):
    """The panel streamer (row panels for C order, column panels for F order)
    accumulates A^T Y / A_J^T Y at a power-of-two scale set by its first
    panel, so tiny fp32 inputs factor like the unit-scale ones."""
    from paper_1706_07191_b200 import SketchConfig
    from paper_1706_07191_b200.rsvd import run_rsvd, run_rsvd_stream
    a = ref_cpu.lowrank_plus_noise(3000, 1200, 20, 1e-3, seed=21, dtype=np.float32)
    omega = ref_cpu.normal_sketch(1200, 30, 0, dtype=np.float32)
    cfg = SketchConfig(20, 10, 2)
    base = run_rsvd(np.asarray(a, order=order), cfg, omega=omega, warn=False)
    st = run_rsvd_stream(np.asarray((a.astype(np.float64) * scale).astype(np.float32),
                                    order=order), cfg, panel=257, nbuf=3, omega=omega,
                         warn=False)
    np.testing.assert_allclose(st.factors.sigma[:20] / scale, base.factors.sigma[:20],
                               rtol=1e-5)
    assert sin_theta(st.factors.U[:, :20], base.factors.U[:, :20]) <= 1e-4


@pytest.mark.parametrize("dtype", [np.float64, np.float32])
@pytest.mark.parametrize("q", [0, 1, 2])
@pytest.mark.parametrize("frac", [0.99, 1.01])
def test_overflow_guard_is_exact_at_threshold(dtype, q, frac):
    """_check_overflow (rsvd.py:84-91): the reference raises iff its
    unnormalised sample peaks above 0.01 * finfo.max.  Inputs scaled to put
    that peak at 0.99x and 1.01x of the threshold: the GPU path (which
    never forms the unnormalised sample in the data's precision) decides
    exactly as the reference does."""
    from paper_1706_07191_b200 import SketchConfig, rsvd_incore
    a = ref_cpu.lowrank_plus_noise(300, 200, 5, 1e-2, seed=8)
    omega = ref_cpu.normal_sketch(200, 10, 0, dtype=np.float64)
    peak1 = float(np.max(np.abs(ref_cpu.power_sample(a, omega, q))))
    lim = 0.01 * float(np.finfo(dtype).max)
    c = (frac * lim / peak1) ** (1.0 / (2 * q + 1))
    ac = (a * c).astype(dtype)
    om = omega.astype(dtype)
    with np.errstate(over="ignore", invalid="ignore"):
        _, ref_fires = ref_cpu.overflow_peak(ref_cpu.power_sample(ac, om, q))
    assert ref_fires == (frac > 1.0)
    cfg = SketchConfig(target_rank=5, oversampling=5, power_exponent=q)
    if ref_fires:
        with pytest.raises(FloatingPointError):
            rsvd_incore(ac, cfg, omega=om)
    else:
        f = rsvd_incore(ac, cfg, omega=om)
        assert np.isfinite(f.sigma).all()
