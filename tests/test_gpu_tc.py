"""The A-streaming products (tcgen05 3xTF32 for fp32, SIMT fp64) against a
float64 torch product: fp32-level accuracy (3xTF32), every layout/transpose,
ragged tiles (M not a multiple of 128, K not a multiple of 16, l not a
multiple of 16)."""

import pytest

pytestmark = pytest.mark.gpu

CASES = [(300, 200, 30), (1000, 777, 120), (130, 129, 5), (4096, 2048, 288),
         (257, 4100, 16), (2049, 100, 64)]


@pytest.mark.parametrize("m,n,l", CASES)
@pytest.mark.parametrize("layout", ["row", "col"])
@pytest.mark.parametrize("trans", [False, True])
def test_fp32_product_accuracy(m, n, l, layout, trans):
    import torch
    from paper_1706_07191_b200.rsvd import sketch_product
    g = torch.Generator(device="cuda").manual_seed(m * 7 + n * 3 + l)
    A = torch.randn(m, n, generator=g, device="cuda", dtype=torch.float32)
    if layout == "col":
        A = A.t().contiguous().t()
    X = torch.randn(m if trans else n, l, generator=g, device="cuda", dtype=torch.float32)
    C = sketch_product(A, X, trans=trans)
    A64 = A.double()
    ref = (A64.t() if trans else A64) @ X.double()
    bound = (A64.abs().t() if trans else A64.abs()) @ X.double().abs()
    err = ((C.double() - ref).abs() / bound.clamp_min(1e-30)).max().item()
    assert err <= 2e-6, err
    C2 = sketch_product(A, X, trans=trans)
    assert torch.equal(C, C2)


@pytest.mark.parametrize("trans", [False, True])
def test_fp64_product(trans):
    import torch
    from paper_1706_07191_b200.rsvd import sketch_product
    g = torch.Generator(device="cuda").manual_seed(5)
    A = torch.randn(700, 300, generator=g, device="cuda", dtype=torch.float64)
    X = torch.randn(700 if trans else 300, 30, generator=g, device="cuda",
                    dtype=torch.float64)
    C = sketch_product(A, X, trans=trans)
    ref = (A.t() if trans else A) @ X
    assert torch.allclose(C, ref, rtol=1e-12, atol=1e-12)
