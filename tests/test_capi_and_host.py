"""CPU-side checks: the C-ABI library builds/loads and exports every symbol
include/brsvd.h declares; host-side logic (config validation, planning, pass
accounting, the .oocm container) behaves like the reference."""

import ctypes
import os
import re
import subprocess
from fractions import Fraction

import numpy as np
import pytest

from tests.conftest import ROOT

HEADER = os.path.join(ROOT, "include", "brsvd.h")


def declared_symbols():
    text = open(HEADER).read()
    return sorted(set(re.findall(r"BRSVD_API\s+[\w\s\*]+?\b(brsvd_\w+)\s*\(", text)))


def test_header_declares_entry_points():
    syms = declared_symbols()
    for s in ("brsvd_rsvd", "brsvd_tsqr", "brsvd_small_svd", "brsvd_gaussian",
              "brsvd_ctx_create", "brsvd_last_error", "brsvd_ialm",
              "brsvd_spectral_norm"):
        assert s in syms, s


def test_library_exports_every_declared_symbol():
    from paper_1706_07191_b200 import build
    so = build.build()
    lib = ctypes.CDLL(so)       # loads without a GPU: cudart is static
    for s in declared_symbols():
        assert hasattr(lib, s), f"{s} not exported"
    nm = subprocess.run(["nm", "-D", "--defined-only", so], capture_output=True,
                        text=True, check=True).stdout
    exported = {line.split()[-1] for line in nm.splitlines() if " T " in line}
    assert set(declared_symbols()) <= exported
    # nothing but the C ABI leaks out
    assert all(s.startswith("brsvd_") for s in exported), sorted(exported)[:10]


def test_library_targets_sm100a():
    from paper_1706_07191_b200 import build
    so = build.build()
    out = subprocess.run(["/usr/local/cuda/bin/cuobjdump", "--list-elf", so],
                         capture_output=True, text=True).stdout
    assert "sm_100a" in out


def test_sketch_config_validation_mirrors_reference():
    from paper_1706_07191_b200 import ConfigError, SketchConfig
    with pytest.raises(ConfigError):
        SketchConfig(target_rank=5, oversampling=5).validate(10, 8)
    with pytest.raises(ConfigError):
        SketchConfig(target_rank=2, power_exponent=99).validate(10, 8)
    with pytest.raises(ConfigError):
        SketchConfig(target_rank=0).validate(10, 8)
    with pytest.raises(ConfigError):
        SketchConfig(target_rank=2, oversampling=-1).validate(10, 8)
    with pytest.raises(ConfigError):
        SketchConfig(target_rank=2, partitions=0).validate(10, 8)
    SketchConfig(target_rank=2, oversampling=2).validate(10, 8)
    assert SketchConfig(target_rank=3, oversampling=4).l == 7


def test_plan_blocks_arithmetic():
    from paper_1706_07191_b200 import BudgetError, plan_blocks
    p = plan_blocks(100, 50, 5, 8)
    assert p.s == 1 and p.blocks == [(0, 100)]
    p = plan_blocks(70, 128, 16, 8, s=7)
    assert p.s == 7 and p.blocks[-1][1] == 70
    budget = 300 * 1024
    p = plan_blocks(256, 512, 13, 8, memory_budget_bytes=budget)
    width = p.n_prime
    assert (512 * width + 3 * 512 * 13 + 2 * width * 13) * 8 <= budget
    assert p.s > 1
    with pytest.raises(BudgetError) as e:
        plan_blocks(256, 512, 13, 8, memory_budget_bytes=1000)
    assert e.value.minimum_feasible > 1000


def test_store_roundtrip_and_accounting(tmp_path):
    from paper_1706_07191_b200 import MatrixStore
    a = np.arange(60, dtype=np.float64).reshape(6, 10)
    st = MatrixStore.from_array(tmp_path / "a.oocm", a)
    assert st.stats.words_read == 0
    np.testing.assert_array_equal(st.read_full(), a)
    np.testing.assert_array_equal(st.read_block(3, 7), a[:, 3:7])
    assert st.stats.block_reads == 2
    assert st.stats.full_passes == Fraction(60 + 24, 60)
    with pytest.raises(IndexError):
        st.read_block(5, 11)
    st.close()
    raw = open(tmp_path / "a.oocm", "rb").read()
    assert raw[:4] == b"OOCM" and len(raw) == 24 + 60 * 8
    # column-major payload
    assert np.frombuffer(raw[24:24 + 16], dtype="<f8").tolist() == [0.0, 10.0]


def test_store_interoperates_with_reference_format(tmp_path):
    """Files written by the reference's MatrixStore load here and vice versa."""
    import sys
    ref_src = "/root/reference/pkg/src"
    if not os.path.isdir(ref_src):
        pytest.skip("reference not mounted")
    sys.path.insert(0, ref_src)
    try:
        import blocksvd as ref
    finally:
        sys.path.remove(ref_src)
    from paper_1706_07191_b200 import MatrixStore
    a = np.random.default_rng(0).standard_normal((9, 4)).astype(np.float32)
    ref.MatrixStore.from_array(tmp_path / "r.oocm", a).close()
    np.testing.assert_array_equal(MatrixStore(tmp_path / "r.oocm").read_full(), a)
    MatrixStore.from_array(tmp_path / "o.oocm", a).close()
    np.testing.assert_array_equal(ref.MatrixStore(tmp_path / "o.oocm").read_full(), a)


def test_shrink_and_rpca_config():
    from paper_1706_07191_b200 import RpcaConfig, shrink
    assert shrink(5.0, 2.0) == 3.0
    assert shrink(-5.0, 2.0) == -3.0
    assert shrink(1.0, 2.0) == 0.0
    np.testing.assert_array_equal(shrink(np.array([[3.0, -0.5], [-2.0, 1.0]]), 1.0),
                                  [[2.0, 0.0], [-1.0, 0.0]])
    with pytest.raises(ValueError):
        shrink(1.0, -0.1)
    for bad in (dict(rho=0.9), dict(tol=0.0), dict(lam=-1.0), dict(mu0=0.0),
                dict(max_iterations=0)):
        with pytest.raises(ValueError):
            RpcaConfig(target_rank=3, **bad).validate()


def test_product_path_fails_loudly_without_library(monkeypatch, tmp_path):
    from paper_1706_07191_b200 import _lib
    monkeypatch.setattr(_lib, "_lib", None)
    with pytest.raises(_lib.BackendUnavailable):
        _lib.load_library(str(tmp_path / "missing.so"))
