"""The persistent CTA-pair tcgen05 product (csrc/tc_stream.cuh, opt-in with
BRSVD_TCS=1; tc3 is the default product kernel) against
a float64 torch product, at shapes that exercise each of its schedules:
stream-K over all resident clusters (many row-tile pairs, tiles split
between two clusters and combined by two atomicAdds), fixed K halves (few
row tiles, long K), whole tiles (short K), the npad buckets up to l = 320,
and K / M tails that are not multiples of the 32-k stage or the 256-row tile
pair.  Results must be fp32-accurate (<= 2e-6 of |A||X|), bit-reproducible
across calls, and agree with the per-tile tc3 kernel (BRSVD_TCS=0) to the
same accuracy."""

import pytest

pytestmark = pytest.mark.gpu

CASES = [(40000, 3001, 288), (33000, 1000, 250), (20000, 2500, 200), (2000, 40000, 288),
         (70000, 290, 120), (300, 100000, 64), (9000, 777, 96), (129, 70000, 30)]


def _product(m, n, l, layout, trans, seed):
    import torch
    g = torch.Generator(device="cuda").manual_seed(seed)
    A = torch.randn(m, n, generator=g, device="cuda", dtype=torch.float32)
    if layout == "col":
        A = A.t().contiguous().t()
    X = torch.randn(m if trans else n, l, generator=g, device="cuda", dtype=torch.float32)
    return A, X


def _rel_err(A, X, C, trans):
    A64 = A.double()
    ref = (A64.t() if trans else A64) @ X.double()
    bound = (A64.abs().t() if trans else A64.abs()) @ X.double().abs()
    return ((C.double() - ref).abs() / bound.clamp_min(1e-30)).max().item()


@pytest.mark.parametrize("m,n,l", CASES)
@pytest.mark.parametrize("layout", ["row", "col"])
@pytest.mark.parametrize("trans", [False, True])
def test_tcs_product(m, n, l, layout, trans, monkeypatch):
    import torch
    from paper_1706_07191_b200.rsvd import sketch_product
    monkeypatch.setenv("BRSVD_TCS", "1")                          # the pair kernel (opt-in)
    A, X = _product(m, n, l, layout, trans, m + 3 * n + l)
    C = sketch_product(A, X, trans=trans)
    assert torch.isfinite(C).all()
    assert _rel_err(A, X, C, trans) <= 2e-6
    assert torch.equal(C, sketch_product(A, X, trans=trans))     # deterministic
    monkeypatch.setenv("BRSVD_TCS", "0")                          # per-tile tc3 kernel
    C3 = sketch_product(A, X, trans=trans)
    assert _rel_err(A, X, C3, trans) <= 2e-6
    scale = (A.abs().double().t() if trans else A.abs().double()) @ X.abs().double()
    assert ((C.double() - C3.double()).abs() / scale).max().item() <= 4e-6
