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


@pytest.mark.parametrize("m,n,l", [(700, 300, 30), (1000, 2999, 1), (4097, 517, 8),
                                   (333, 5000, 13), (2048, 1024, 20), (513, 700, 48),
                                   (1500, 1300, 64), (300, 200, 100)])
@pytest.mark.parametrize("layout", ["row", "col"])
@pytest.mark.parametrize("trans", [False, True])
def test_fp64_product(m, n, l, layout, trans):
    """fp64 skinny products (kc/mc kernels, l <= 64; generic tiles above),
    both storage orders, ragged sizes, deterministic."""
    import torch
    from paper_1706_07191_b200.rsvd import sketch_product
    g = torch.Generator(device="cuda").manual_seed(m + 3 * n + 7 * l)
    A = torch.randn(m, n, generator=g, device="cuda", dtype=torch.float64)
    if layout == "col":
        A = A.t().contiguous().t()
    X = torch.randn(m if trans else n, l, generator=g, device="cuda", dtype=torch.float64)
    C = sketch_product(A, X, trans=trans)
    ref = (A.t() if trans else A) @ X
    bound = (A.abs().t() if trans else A.abs()) @ X.abs()
    err = ((C - ref).abs() / bound).max().item()
    assert err <= 1e-14, err
    assert torch.equal(C, sketch_product(A, X, trans=trans))


@pytest.mark.parametrize("trans", [False, True])
@pytest.mark.parametrize("h16", ["1"])
def test_fp32_product_dynamic_range(trans, h16, monkeypatch):
    """Rows and sketch columns spanning 1e-38..1e25 (plus zero and subnormal
    rows): the fp16-split path scales each row/column by a power of two, so
    every output entry stays accurate relative to its own |A||X| bound.  (The
    unscaled 3xTF32 path behind BRSVD_TC_H16=0 is a diagnostic switch only: its
    low-part terms underflow for tiny-magnitude rows, so it is not held to
    this.)"""
    import torch
    from paper_1706_07191_b200.rsvd import sketch_product
    monkeypatch.setenv("BRSVD_TC_H16", h16)
    m, n, l = 1024, 640, 24
    g = torch.Generator(device="cuda").manual_seed(11)
    A = torch.randn(m, n, generator=g, device="cuda", dtype=torch.float64)
    exps = torch.linspace(-38, 25, m, device="cuda", dtype=torch.float64)
    A = A * torch.pow(10.0, exps)[:, None]
    A[5] = 0
    A[7] = A[7].sign() * 1e-41          # subnormal fp32 row
    if trans:
        A = A.t().contiguous()
    A = A.float()
    X = torch.randn(A.shape[0] if trans else A.shape[1], l, generator=g,
                    device="cuda", dtype=torch.float64)
    X = (X * torch.pow(10.0, torch.linspace(-20, 6, l, device="cuda",
                                            dtype=torch.float64))[None, :]).float()
    C = sketch_product(A, X, trans=trans)
    A64, X64 = A.double(), X.double()
    ref = (A64.t() if trans else A64) @ X64
    bound = (A64.abs().t() if trans else A64.abs()) @ X64.abs()
    ok = bound > 1e-36                   # fp32-representable outputs
    assert torch.isfinite(C).all()
    err = ((C.double() - ref).abs() / bound.clamp_min(1e-300))[ok].max().item()
    assert err <= 2e-6, err


@pytest.mark.parametrize("m,n", [(1024, 640), (1027, 333), (4096, 130), (3, 5000)])
@pytest.mark.parametrize("layout", ["row", "col"])
def test_absmax_rows_cols(m, n, layout):
    """Row/column maxima of |A| (the fp16-split scales): vectorised and scalar
    kernels, both storage orders, ragged sizes, a NaN-free exact match."""
    import torch
    from paper_1706_07191_b200.distributed import GpuOps
    g = torch.Generator(device="cuda").manual_seed(m * 5 + n)
    A = torch.randn(m, n, generator=g, device="cuda", dtype=torch.float32)
    A[m // 2] *= 1e20
    A[:, n // 3] *= 1e-30
    if layout == "col":
        A = A.t().contiguous().t()
    rmax, cmax = GpuOps().absmax(A)
    assert torch.equal(rmax, A.abs().amax(dim=1))
    assert torch.equal(cmax, A.abs().amax(dim=0))


@pytest.mark.parametrize("m,n,l", [(1, 1, 1), (1, 300, 5), (300, 1, 5), (17, 33, 64),
                                   (129, 17, 2), (5, 4000, 12)])
@pytest.mark.parametrize("layout", ["row", "col", "odd_ld"])
@pytest.mark.parametrize("trans", [False, True])
def test_fp64_product_edges(m, n, l, layout, trans):
    """fp64 skinny products at degenerate and ragged shapes, and with an odd
    leading dimension (not 16-byte aligned rows: the generic tiled kernel)."""
    import torch
    from paper_1706_07191_b200.rsvd import sketch_product
    g = torch.Generator(device="cuda").manual_seed(m * 131 + n * 7 + l)
    if layout == "odd_ld":
        stride = n + 1 if (n + 1) % 2 else n + 2        # an odd row stride
        A = torch.randn(m, stride, generator=g, device="cuda", dtype=torch.float64)[:, :n]
    else:
        A = torch.randn(m, n, generator=g, device="cuda", dtype=torch.float64)
        if layout == "col":
            A = A.t().contiguous().t()
    X = torch.randn(m if trans else n, l, generator=g, device="cuda", dtype=torch.float64)
    C = sketch_product(A, X, trans=trans)
    ref = (A.t() if trans else A) @ X
    bound = (A.abs().t() if trans else A.abs()) @ X.abs()
    err = ((C - ref).abs() / bound.clamp_min(1e-300)).max().item()
    assert err <= 1e-14, err


@pytest.mark.parametrize("ksplit", ["1", "2", "3", "4"])
@pytest.mark.parametrize("l", [200, 288])
@pytest.mark.parametrize("layout,trans", [("row", False), ("col", True), ("col", False)])
def test_single_chunk_pair_ksplits(ksplit, l, layout, trans, monkeypatch):
    """The single-chunk CTA-pair product (160 < l <= 288) with 1-4 K-splits
    forced (BRSVD_TCW_KSPLIT): every split count meets the fp32-level bound,
    and a split count > 1 (partials summed in split order) is deterministic."""
    import torch
    from paper_1706_07191_b200.rsvd import sketch_product
    monkeypatch.setenv("BRSVD_TCW_KSPLIT", ksplit)
    m, n = (16384, 1000) if trans else (1000, 16384)
    g = torch.Generator(device="cuda").manual_seed(l + 11 * int(ksplit))
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
    assert torch.equal(C, sketch_product(A, X, trans=trans))
