"""Sampled fp16-split scales (LazyScales, csrc/pipeline.cuh).

The device-resident fp32 path no longer reads all of A for the per-row /
per-column scales of the fp16-split products: the first product of each
orientation runs on sampled maxima and records the exact ones, and a flagged
line re-runs that product on the exact scales.  These tests pin both
branches against the eager path (BRSVD_LAZY_SCALES=0, one absmax pass up
front, the round-1 behaviour) and against the CPU oracle:
  * inputs whose largest entries hide from the sample (a spike outside every
    sampled line, a row that is zero at every sampled position) take the
    re-run in both orientations, which then computes with exactly the eager
    path's scales -- the factors are bit-identical;
  * ordinary inputs keep the sampled scales, which serve the same 22-bit
    split, so the factors agree with the eager ones to fp32 rounding and with
    the oracle to the north star's fp32 tolerances.
"""

import os

import numpy as np
import pytest

from oracle import ref_cpu

pytestmark = pytest.mark.gpu

K, P = 200, 32          # l = 232: the single-chunk pair kernel


def _run(a_dev, q, omega, lazy):
    from paper_1706_07191_b200 import SketchConfig, rsvd_incore
    old = os.environ.get("BRSVD_LAZY_SCALES")
    os.environ["BRSVD_LAZY_SCALES"] = "1" if lazy else "0"
    try:
        f = rsvd_incore(a_dev, SketchConfig(K, P, q), omega=omega)
    finally:
        if old is None:
            del os.environ["BRSVD_LAZY_SCALES"]
        else:
            os.environ["BRSVD_LAZY_SCALES"] = old
    return (f.sigma.cpu().numpy(), f.U.cpu().numpy(), f.Vt.cpu().numpy())


def _device(a, order):
    import torch
    if order == "C":
        return torch.as_tensor(np.ascontiguousarray(a), device="cuda")
    return torch.as_tensor(np.ascontiguousarray(a.T), device="cuda").t()


def _sampled(n):
    """Positions along a line of length n that the sample reads: every 32nd
    line whole (the contiguous index) and chunks [4096 k, 4096 k + 128) of
    every line (the outer index) -- tc::amax_sample_outer_kernel."""
    chunks = np.zeros(n, dtype=bool)
    for c in range(0, n, 4096):
        chunks[c:c + 128] = True
    every32 = np.zeros(n, dtype=bool)
    every32[::32] = True
    return chunks | every32


def _hidden_extremes(a):
    """A spike at (1000, 1000), which no sampled line or chunk of either
    orientation reads, plus row 300 / column 700 zero at every sampled
    position and 1e-6 smaller elsewhere (the sampled maximum is 0)."""
    a = a.copy()
    big = float(np.abs(a).max())
    a[1000, 1000] = 1e5 * big
    a[300, :] *= 1e-6
    a[300, _sampled(a.shape[1])] = 0.0
    a[:, 700] *= 1e-6
    a[_sampled(a.shape[0]), 700] = 0.0
    return a


@pytest.mark.parametrize("order", ["C", "F"])
@pytest.mark.parametrize("q", [0, 2])
def test_rerun_on_exact_scales_is_bit_identical(order, q):
    a = _hidden_extremes(ref_cpu.lowrank_plus_noise(2048, 1792, 220, 1e-3, seed=11,
                                                    dtype=np.float32))
    omega = ref_cpu.normal_sketch(a.shape[1], K + P, 0, dtype=np.float32)
    ad = _device(a, order)
    s_l, u_l, v_l = _run(ad, q, omega, lazy=True)
    s_e, u_e, v_e = _run(ad, q, omega, lazy=False)
    assert np.array_equal(s_l, s_e)
    assert np.array_equal(u_l, u_e) and np.array_equal(v_l, v_e)


@pytest.mark.parametrize("order", ["C", "F"])
def test_sampled_scales_match_eager_and_oracle(order):
    a = ref_cpu.lowrank_plus_noise(2048, 1792, 220, 1e-3, seed=12, dtype=np.float32)
    omega = ref_cpu.normal_sketch(a.shape[1], K + P, 0, dtype=np.float32)
    ad = _device(a, order)
    s_l, u_l, _ = _run(ad, 2, omega, lazy=True)
    s_e, u_e, _ = _run(ad, 2, omega, lazy=False)
    np.testing.assert_allclose(s_l[:K], s_e[:K], rtol=1e-6)
    ref = ref_cpu.randomized_svd(a, K, P, 2, seed=0, omega=omega)
    np.testing.assert_allclose(s_l[:K], ref["sigma"][:K], rtol=1e-5)
    qa, _ = np.linalg.qr(u_l[:, :K].astype(np.float64))
    qb, _ = np.linalg.qr(ref["U"][:, :K].astype(np.float64))
    assert np.linalg.norm(qa - qb @ (qb.T @ qa), 2) <= 1e-3
