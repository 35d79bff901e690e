"""Pin the CPU oracle (oracle/ref_cpu.py) to the reference's own outputs.

tests/golden/*.npz were produced by running the reference package
(oracle/make_golden.py).  The oracle must reproduce them to rounding before
it is trusted as the checker of the GPU path.  CPU only.
"""

import os

import numpy as np
import pytest

from oracle import ref_cpu
from tests.conftest import GOLDEN


def load(name):
    return np.load(os.path.join(GOLDEN, name))


RSVD_CASES = ["c1small_f64", "lr4_q0", "lr4_q1", "lr4_q2", "exact_rank8", "f32_rank48",
              "wide_f64", "decay_f64"]


@pytest.mark.parametrize("case", RSVD_CASES)
def test_rsvd_matches_reference(case):
    g = load(f"rsvd_{case}.npz")
    a = g["a"]
    k, p, q, seed = int(g["k"]), int(g["p"]), int(g["q"]), int(g["seed"])
    out = ref_cpu.randomized_svd(a, k, p, q, seed)
    # Omega regenerated from the seed reproduces the reference's exactly.
    assert np.array_equal(out["omega"], g["omega"])
    tol = 1e-10 if a.dtype == np.float64 else 1e-5
    np.testing.assert_allclose(out["sigma"][:k], g["sigma"][:k], rtol=tol)
    # same canonical signs -> same leading vectors
    atol = 1e-7 if a.dtype == np.float64 else 1e-3
    np.testing.assert_allclose(out["U"][:, :k], g["U"][:, :k], atol=atol)
    np.testing.assert_allclose(out["Vt"][:k], g["Vt"][:k], atol=atol)
    err = ref_cpu.frob_rel_error(a, out["U"], out["sigma"], out["Vt"])
    assert abs(err - float(g["relerr"])) <= 1e-6 * max(1.0, float(g["relerr"]))


def test_rank_warnings_match_reference():
    g = load("rsvd_exact_rank8.npz")
    out = ref_cpu.randomized_svd(g["a"], 8, 4, 1, 0)
    assert [out["rank_y"], out["rank_b"]] == list(g["warned_ranks"])


def test_gaussian_stream_matches_reference():
    g = load("gaussian.npz")
    assert np.array_equal(ref_cpu.normal_sketch(50, 7, 123, 4), g["g"])
    assert np.array_equal(ref_cpu.normal_sketch(20, 7, 123, 4, row_offset=30), g["g_off"])
    assert np.array_equal(g["g"][30:], g["g_off"])
    assert np.array_equal(ref_cpu.normal_sketch(40, 5, 9, dtype=np.float32), g["g32"])


def test_tsqr_matches_reference():
    g = load("tsqr.npz")
    q, r, rank = ref_cpu.orthonormal_range(g["y"], block_rows=100)
    np.testing.assert_allclose(q, g["q"], atol=1e-12)
    np.testing.assert_allclose(r, g["r"], atol=1e-10)
    _, _, rank_def = ref_cpu.orthonormal_range(g["y_def"])
    assert rank_def == int(g["rank_def"]) == 2


def test_small_svd_matches_reference():
    g = load("small_svd.npz")
    w, s, vt, _ = ref_cpu.core_svd(g["b"])
    np.testing.assert_allclose(s, g["sigma"], rtol=1e-12)
    np.testing.assert_allclose(np.abs(w), np.abs(g["W"]), atol=1e-10)
    _, sd, _, rank = ref_cpu.core_svd(g["b_def"])
    assert rank == 2
    np.testing.assert_allclose(sd[:2], g["sigma_def"][:2], rtol=1e-12)


def test_naive_ooc_matches_reference():
    g = load("naive_ooc.npz")
    out = ref_cpu.randomized_svd_blocked(g["a"], 5, 10, 2, 3, partitions=5)
    np.testing.assert_allclose(out["sigma"][:5], g["sigma"][:5], rtol=1e-10)
    assert float(g["passes"]) == 6.0   # 2(q+1), rsvd.py:218-224


def test_rpca_matches_reference():
    g = load("rpca_planted.npz")
    out = ref_cpu.ialm(g["M"], 10, 10, 1)
    assert out["iterations"] == int(g["iterations"])
    np.testing.assert_allclose(out["residuals"], g["residuals"], rtol=1e-6)
    np.testing.assert_allclose(out["mus"], g["mus"], rtol=1e-12)
    np.testing.assert_allclose(out["L"], g["L"], atol=1e-8)
    assert abs(ref_cpu.power_norm(g["M"]) - float(g["norm2"])) <= 1e-9 * float(g["norm2"])


def test_shrink_piecewise():
    x = np.array([5.0, -5.0, 1.0, 0.0])
    np.testing.assert_array_equal(ref_cpu.soft_threshold(x, 2.0), [3.0, -3.0, 0.0, 0.0])


@pytest.mark.parametrize("name", ["brsvd_paper_s4_q2.npz", "brsvd_paper_s3_q1.npz"])
def test_paper_mode_matches_reference_brsvd_run(name):
    """brsvd_run with s > 1, q >= 1: the per-block power iteration (two passes)."""
    g = load(name)
    k, p, q = int(g["k"]), int(g["p"]), int(g["q"])
    blocks = [tuple(b) for b in g["blocks"]]
    assert len(blocks) == int(g["s"])
    out = ref_cpu.randomized_svd_paper(g["a"], k, p, q, blocks, seed=int(g["seed"]))
    np.testing.assert_allclose(out["sigma"][:k], g["sigma"][:k], rtol=1e-10)
    assert float(g["passes"]) == 2.0   # rsvd.py:188-193
    # a different approximation from the global iteration
    glob = ref_cpu.randomized_svd(g["a"], k, p, q, seed=int(g["seed"]), omega=g["omega"])
    assert np.max(np.abs(glob["sigma"][:k] - g["sigma"][:k]) / g["sigma"][:k]) > 1e-8


def test_rpca_out_of_core_branch_matches_reference():
    """rpca.py:216-304: store input above the budget; the inner SVD is the
    per-block brsvd_run over the budget's column blocks."""
    g = load("rpca_ooc.npz")
    blocks = [(int(a), int(b)) for a, b in g["blocks"]]
    out = ref_cpu.ialm(g["M"], 10, 10, 1, blocks=blocks)
    assert out["iterations"] == int(g["iterations"])
    np.testing.assert_allclose(out["residuals"], g["residuals"], rtol=1e-6)
    np.testing.assert_allclose(out["L"], g["L"], atol=1e-8)


def test_naive_ooc_sketch_and_factors_match_reference():
    """rsvd_naive_ooc (rsvd.py:218-284): the stored global sketch is the
    per-block slices' union (kernels.py:98-118 row_offset) and the oracle's
    blocked global iteration reproduces the reference's factors."""
    g = load("naive_ooc.npz")
    k, p, q, s, seed = (int(g[x]) for x in ("k", "p", "q", "s", "seed"))
    assert np.array_equal(ref_cpu.normal_sketch(100, k + p, seed), g["omega"])
    out = ref_cpu.randomized_svd_blocked(g["a"], k, p, q, seed, partitions=s)
    np.testing.assert_allclose(out["sigma"][:k], g["sigma"][:k], rtol=1e-10)
    np.testing.assert_allclose(out["U"][:, :k], g["U"][:, :k], atol=1e-8)
    assert float(g["passes"]) == 2 * (q + 1) and int(g["block_reads"]) == 2 * (q + 1) * s


@pytest.mark.parametrize("s,q", [(1, 1), (3, 2)])
def test_range_finder_matches_reference(s, q):
    g = load("range_finder.npz")
    blocks = g[f"blocks_s{s}_q{q}"]
    Q, _ = ref_cpu.range_basis_paper(g["a"], 6, 6, q, blocks, seed=11)
    assert np.array_equal(ref_cpu.normal_sketch(180, 12, 11), g["omega"])
    Qr = g[f"Q_s{s}_q{q}"]
    # same Householder tree: the leading (numerically determined) columns
    # agree to rounding; the trailing ones span noise-floor directions of the
    # sample and differ at its rounding level (1e-5 for s = 1, q = 1)
    np.testing.assert_allclose(Q[:, :8], Qr[:, :8], atol=1e-12)
    assert np.linalg.norm(Q[:, :6] @ Q[:, :6].T - Qr[:, :6] @ Qr[:, :6].T) <= 1e-12


def test_video_slice_input_is_the_referenced_matrix():
    """The config-5 slice golden regenerates M from ref_cpu.video_matrix; its
    checksums pin that generator (numpy default_rng) to what the reference
    was run on."""
    g = load("rpca_video_slice.npz")
    M = ref_cpu.video_matrix(int(g["width"]), int(g["height"]), int(g["frames"]),
                             seed=int(g["seed"]))
    assert M.sum() == float(g["M_sum"]) and float((M * M).sum()) == float(g["M_sq"])
    assert np.array_equal(ref_cpu.normal_sketch(M.shape[1], 20, 0), g["omega"])
    assert int(g["iterations"]) == len(g["residuals"]) and bool(g["converged"])
