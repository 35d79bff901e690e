"""Debug: dynamic-range product, tcs vs tc3 (prints the worst entries)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_1706_07191_b200.rsvd import sketch_product
for trans in (False, True):
    m, n, l = 1024, 640, 24
    g = torch.Generator(device="cuda").manual_seed(11)
    A = torch.randn(m, n, generator=g, device="cuda", dtype=torch.float64)
    exps = torch.linspace(-38, 25, m, device="cuda", dtype=torch.float64)
    A = A * torch.pow(10.0, exps)[:, None]
    A[5] = 0
    A[7] = A[7].sign() * 1e-41
    if trans:
        A = A.t().contiguous()
    A = A.float()
    X = torch.randn(A.shape[0] if trans else A.shape[1], l, generator=g, device="cuda", dtype=torch.float64)
    X = (X * torch.pow(10.0, torch.linspace(-20, 6, l, device="cuda", dtype=torch.float64))[None, :]).float()
    A64, X64 = A.double(), X.double()
    ref = (A64.t() if trans else A64) @ X64
    bound = (A64.abs().t() if trans else A64.abs()) @ X64.abs()
    ok = bound > 1e-36
    for tcs in ("1", "0"):
        os.environ["BRSVD_TCS"] = tcs
        C = sketch_product(A, X, trans=trans)
        e = ((C.double() - ref).abs() / bound.clamp_min(1e-300))
        e[~ok] = 0
        i = int(e.argmax())
        r, c = i // l, i % l
        print(f"trans {trans} tcs {tcs}: max err {e.max().item():.3e} at row {r} col {c}: C {C[r,c].item():.6e} ref {ref[r,c].item():.6e} bound {bound[r,c].item():.3e}; rows>1e-6 err: {(e.amax(dim=1) > 1e-6).nonzero().flatten()[:20].tolist()}")
