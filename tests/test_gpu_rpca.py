"""GPU robust PCA (brsvd_ialm) against the reference's results and its own
test properties (tests/test_rpca.py of the reference)."""

import os

import numpy as np
import pytest

from oracle import ref_cpu
from tests.conftest import GOLDEN

pytestmark = pytest.mark.gpu


def planted(m=200, n=200, rank=5, density=0.05, seed=0):
    rng = np.random.default_rng(seed)
    L0 = rng.standard_normal((m, rank)) @ rng.standard_normal((rank, n))
    mask = rng.random((m, n)) < density
    S0 = np.zeros((m, n))
    S0[mask] = rng.choice([-1.0, 1.0], size=int(mask.sum())) * np.max(np.abs(L0))
    return L0, S0, mask


def test_planted_matches_reference_golden():
    from paper_1706_07191_b200 import RpcaConfig, ialm_rpca
    g = np.load(os.path.join(GOLDEN, "rpca_planted.npz"))
    res = ialm_rpca(g["M"], RpcaConfig(target_rank=10, tol=1e-7), omega=g["omega"])
    assert res.converged
    assert abs(res.iterations - int(g["iterations"])) <= 1
    k = min(res.iterations, int(g["iterations"])) - 1
    # same sketch as the reference: same trajectory (the spectral-norm start
    # vector differs, which moves mu0 by ~1e-10 relative)
    np.testing.assert_allclose(res.residual_history[:k], g["residuals"][:k], rtol=1e-4)
    np.testing.assert_allclose([h["mu"] for h in res.history][:k], g["mus"][:k],
                               rtol=1e-9)
    rel = np.linalg.norm(res.L - g["L"]) / np.linalg.norm(g["L"])
    assert rel <= 1e-6, rel
    assert np.linalg.norm(res.L - g["L0"]) / np.linalg.norm(g["L0"]) <= 1e-4
    support = np.abs(res.S) > 1e-6
    assert (support & g["mask"]).sum() / g["mask"].sum() >= 0.95


def test_against_live_oracle_fp32_column_major():
    from paper_1706_07191_b200 import RpcaConfig, ialm_rpca
    L0, S0, _ = planted(m=300, n=120, seed=3)
    M = np.asfortranarray((L0 + S0).astype(np.float32))
    ref = ref_cpu.ialm(M, 10, 10, 1, tol=1e-5)
    res = ialm_rpca(M, RpcaConfig(target_rank=10, tol=1e-5))
    assert res.L.dtype == np.float32 and res.L.flags.f_contiguous
    assert abs(res.iterations - ref["iterations"]) <= 1
    rel = np.linalg.norm(res.L - ref["L"]) / np.linalg.norm(ref["L"])
    assert rel <= 1e-4, rel


def test_no_corruption_gives_null_sparse():
    from paper_1706_07191_b200 import RpcaConfig, ialm_rpca
    rng = np.random.default_rng(5)
    M = rng.standard_normal((120, 3)) @ rng.standard_normal((3, 80))
    res = ialm_rpca(M, RpcaConfig(target_rank=5, tol=1e-7))
    assert res.converged
    assert np.linalg.norm(res.S) / np.linalg.norm(M) <= 1e-6
    assert np.linalg.norm(res.L - M) / np.linalg.norm(M) <= 1e-6


def test_mu_schedule_history_and_flags():
    from paper_1706_07191_b200 import RpcaConfig, ialm_rpca
    L0, S0, _ = planted(seed=6)
    res = ialm_rpca(L0 + S0, RpcaConfig(target_rank=10, tol=1e-7, mu0=0.01, rho=1.5))
    mus = [h["mu"] for h in res.history]
    assert np.allclose(mus, [0.01 * 1.5 ** i for i in range(len(mus))])
    assert res.residual_history[-1] < 1e-7
    assert [h["i"] for h in res.history] == list(range(1, res.iterations + 1))
    assert len(res.to_json_lines().splitlines()) == res.iterations
    res = ialm_rpca(L0 + S0, RpcaConfig(target_rank=10, tol=1e-7, max_iterations=3))
    assert not res.converged and res.iterations == 3


def test_large_lambda_kills_sparse_term_and_determinism():
    from paper_1706_07191_b200 import RpcaConfig, ialm_rpca
    L0, S0, _ = planted(seed=8)
    res = ialm_rpca(L0 + S0, RpcaConfig(target_rank=10, lam=1e6, tol=1e-7,
                                        max_iterations=20))
    assert np.count_nonzero(res.S) == 0
    cfg = RpcaConfig(target_rank=10, tol=1e-7, master_seed=5)
    r1, r2 = ialm_rpca(L0 + S0, cfg), ialm_rpca(L0 + S0, cfg)
    assert r1.iterations == r2.iterations
    assert np.array_equal(r1.L, r2.L) and np.array_equal(r1.S, r2.S)


def test_zero_input_rejected():
    from paper_1706_07191_b200 import RpcaConfig, ialm_rpca
    with pytest.raises(ValueError):
        ialm_rpca(np.zeros((10, 10)), RpcaConfig(target_rank=2, oversampling=2))


def test_spectral_norm_known_answers():
    from paper_1706_07191_b200 import spectral_norm_estimate
    assert abs(spectral_norm_estimate(np.diag([3.0, 1.0])) - 3.0) <= 1e-6
    rng = np.random.default_rng(2)
    u = rng.standard_normal(50)
    u *= 2.0 / np.linalg.norm(u)
    v = rng.standard_normal(30)
    v *= 3.0 / np.linalg.norm(v)
    assert abs(spectral_norm_estimate(np.outer(u, v)) - 6.0) <= 1e-6
    a = rng.standard_normal((100, 80))
    s1 = np.linalg.svd(a, compute_uv=False)[0]
    assert abs(spectral_norm_estimate(a) - s1) <= 0.01 * s1
    assert abs(spectral_norm_estimate(np.asfortranarray(a)) - spectral_norm_estimate(a)) \
        <= 1e-8 * s1
    with pytest.warns(UserWarning, match="zero matrix"):
        assert spectral_norm_estimate(np.zeros((4, 4))) == 0.0


@pytest.mark.parametrize("dtype", [np.float64, np.float32])
def test_spectral_norm_matches_oracle_with_reference_start(dtype):
    """spectral_norm_estimate (rpca.py:72-100) from the reference's own start
    vector (gaussian_matrix(n, 1, seed, stream_index=7)) follows the
    reference's power iteration: a random (slow-converging) matrix agrees with
    the oracle to its stopping tolerance, not just to the 1 % of two different
    starts."""
    from oracle import ref_cpu
    from paper_1706_07191_b200 import spectral_norm_estimate
    rng = np.random.default_rng(31)
    a = rng.standard_normal((400, 300)).astype(dtype)
    v0 = ref_cpu.normal_sketch(300, 1, 5, 7, dtype=dtype)[:, 0]
    ref = ref_cpu.power_norm(a, seed=5)
    got = spectral_norm_estimate(a, seed=5, start=v0)
    assert abs(got - ref) <= (1e-9 if dtype == np.float64 else 1e-5) * ref
    got_c = spectral_norm_estimate(np.asfortranarray(a), seed=5, start=v0)
    assert abs(got_c - got) <= 1e-12 * ref


def test_store_paths(tmp_path):
    from paper_1706_07191_b200 import MatrixStore, RpcaConfig, ialm_rpca
    L0, S0, _ = planted(m=80, n=200, seed=12)
    M = L0 + S0
    st = MatrixStore.from_array(tmp_path / "m.oocm", M)
    res = ialm_rpca(st, RpcaConfig(target_rank=10, tol=1e-7, memory_budget_bytes=1 << 30))
    assert isinstance(res.L, np.ndarray) and res.converged
    res_ooc = ialm_rpca(st, RpcaConfig(target_rank=10, tol=1e-7,
                                       memory_budget_bytes=60_000))
    assert isinstance(res_ooc.L, MatrixStore) and res_ooc.converged
    L, S = res_ooc.L.read_full(), res_ooc.S.read_full()
    assert np.linalg.norm(L + S - M) / np.linalg.norm(M) <= 1e-6
    st.close()


def test_device_tensor_input_stays_on_device():
    import torch
    from paper_1706_07191_b200 import RpcaConfig, ialm_rpca
    L0, S0, _ = planted(m=160, n=90, seed=4)
    M = torch.as_tensor(L0 + S0, device="cuda")
    res = ialm_rpca(M, RpcaConfig(target_rank=10, tol=1e-7))
    assert res.L.is_cuda and res.converged
    res_h = ialm_rpca(L0 + S0, RpcaConfig(target_rank=10, tol=1e-7))
    np.testing.assert_allclose(res.L.cpu().numpy(), res_h.L, atol=1e-9)


@pytest.mark.parametrize("stream", [False, True])
def test_out_of_core_branch_matches_reference(tmp_path, stream):
    """Store input above memory_budget_bytes: the reference's out-of-core
    branch (rpca.py:216-304) runs brsvd_run per budget block in each
    iteration; ours uses the same per-block inner SVD (brsvd_ialm_blocked) and
    returns MatrixStore results like the reference.  stream=True: M, S, Y
    host-resident and streamed block by block every pass (brsvd_ialm_stream);
    stream=False: the iterates held in HBM."""
    from paper_1706_07191_b200 import MatrixStore, RpcaConfig, ialm_rpca
    g = np.load(os.path.join(GOLDEN, "rpca_ooc.npz"))
    st = MatrixStore.from_array(tmp_path / "m.oocm", g["M"])
    res = ialm_rpca(st, RpcaConfig(target_rank=10, tol=1e-7,
                                   memory_budget_bytes=int(g["budget"])),
                    omega=g["omega"], stream=stream)
    assert isinstance(res.L, MatrixStore) and isinstance(res.S, MatrixStore)
    assert res.converged
    assert abs(res.iterations - int(g["iterations"])) <= 1
    k = min(res.iterations, int(g["iterations"])) - 1
    np.testing.assert_allclose(res.residual_history[:k], g["residuals"][:k], rtol=1e-4)
    L = res.L.read_full()
    rel = np.linalg.norm(L - g["L"]) / np.linalg.norm(g["L"])
    assert rel <= 1e-6, rel


def test_streamed_ooc_file_backed_matches_pinned(tmp_path):
    """A store beyond host RAM streams M from its memory map and keeps S, Y,
    L in file-backed maps (pinned=False); same iteration as the pinned path."""
    from paper_1706_07191_b200 import MatrixStore, RpcaConfig, ialm_rpca
    L0, S0, _ = planted(m=500, n=180, seed=14)
    st = MatrixStore.from_array(tmp_path / "m.oocm", L0 + S0)
    cfg = RpcaConfig(target_rank=8, tol=1e-7, memory_budget_bytes=(L0.nbytes // 3))
    a = ialm_rpca(st, cfg, stream=True, pinned=True)
    b = ialm_rpca(st, cfg, stream=True, pinned=False)
    assert a.iterations == b.iterations and b.converged
    np.testing.assert_allclose(b.residual_history, a.residual_history, rtol=1e-12)
    np.testing.assert_array_equal(b.L.read_full(), a.L.read_full())
    np.testing.assert_array_equal(b.S.read_full(), a.S.read_full())


def test_streamed_ooc_matches_resident_blocked(tmp_path):
    """The host-streamed IALM and the HBM-resident blocked IALM run the same
    iteration (same plan, same inner SVD semantics): identical iteration
    count, residual history within rounding, L and S within 1e-9."""
    from paper_1706_07191_b200 import MatrixStore, RpcaConfig, ialm_rpca
    L0, S0, _ = planted(m=700, n=260, seed=12)
    st = MatrixStore.from_array(tmp_path / "m.oocm", L0 + S0)
    cfg = RpcaConfig(target_rank=8, tol=1e-7, memory_budget_bytes=(L0.nbytes // 3))
    a = ialm_rpca(st, cfg, stream=False)
    b = ialm_rpca(st, cfg, stream=True)
    assert a.iterations == b.iterations and a.converged and b.converged
    np.testing.assert_allclose(b.residual_history, a.residual_history, rtol=1e-6)
    for x, y in ((a.L, b.L), (a.S, b.S)):
        np.testing.assert_allclose(y.read_full(), x.read_full(), atol=1e-9)
