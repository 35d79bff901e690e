"""Fused residual kernel (brsvd_residual) behind relative_frobenius_error
(rsvd.py:396-432) against the CPU oracle (oracle/ref_cpu.frob_rel_error).

Tolerances: fp64 inputs agree to 1e-10 relative on the error value; fp32
inputs (the reconstruction is formed in fp32, sums of squares in fp64) to
1e-4 relative, the north star's tolerance for the relative error."""

import os

import numpy as np
import pytest

from oracle import ref_cpu

pytestmark = pytest.mark.gpu


def _factors(a, k, p, q):
    from paper_1706_07191_b200 import SketchConfig, rsvd_incore
    return rsvd_incore(a, SketchConfig(target_rank=k, oversampling=p, power_exponent=q))


@pytest.mark.parametrize("layout", ["C", "F"])
def test_residual_f64_config1_shape(layout):
    from paper_1706_07191_b200 import relative_frobenius_error
    a = ref_cpu.lowrank_plus_noise(10000, 2000, 20, 1e-3, seed=3)
    a = np.asarray(a, order=layout)
    f = _factors(a, 20, 10, 2)
    ref = ref_cpu.frob_rel_error(a, f.U, f.sigma, f.Vt)
    got = relative_frobenius_error(a, f)
    assert abs(got - ref) <= 1e-10 * ref


def test_residual_f32_and_ragged_tiles():
    from paper_1706_07191_b200 import relative_frobenius_error
    a = ref_cpu.lowrank_plus_noise(3001, 1537, 40, 1e-2, seed=5).astype(np.float32)
    f = _factors(a, 40, 8, 1)
    ref = ref_cpu.frob_rel_error(a.astype(np.float64), f.U.astype(np.float64),
                                 f.sigma.astype(np.float64), f.Vt.astype(np.float64))
    got = relative_frobenius_error(a, f)
    assert abs(got - ref) <= 1e-4 * ref


def test_residual_store_blocks_match_in_memory(tmp_path):
    from paper_1706_07191_b200 import MatrixStore, relative_frobenius_error
    a = ref_cpu.lowrank_plus_noise(700, 333, 12, 1e-3, seed=9)
    f = _factors(a, 12, 6, 1)
    store = MatrixStore.create(os.path.join(tmp_path, "a.oocm"), 700, 333, np.float64)
    store.write_block(0, 333, a)
    whole = relative_frobenius_error(a, f)
    for bw in (1, 50, 333):
        blk = relative_frobenius_error(store, f, block_width=bw)
        assert abs(blk - whole) <= 1e-12 * whole
    assert abs(whole - ref_cpu.frob_rel_error(a, f.U, f.sigma, f.Vt)) <= 1e-10 * whole


def test_residual_zero_and_exact():
    from paper_1706_07191_b200 import relative_frobenius_error
    from paper_1706_07191_b200.kernels import SvdFactors
    z = np.zeros((64, 32))
    f = SvdFactors(U=np.zeros((64, 4)), sigma=np.zeros(4), Vt=np.zeros((4, 32)),
                   target_rank=4, effective_l=4)
    assert relative_frobenius_error(z, f) == 0.0
    rng = np.random.default_rng(2)
    a = rng.standard_normal((256, 3)) @ rng.standard_normal((3, 96))
    f = _factors(a, 3, 5, 1)
    assert relative_frobenius_error(a, f) <= 1e-12
