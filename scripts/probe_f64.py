"""Timing of the fp64 A-streaming products at the C5 / C1 shapes."""
import os, sys, torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1706_07191_b200.rsvd import sketch_product
for (m, n, l) in [(76800, 20000, 20), (10000, 2000, 30)]:
    A = torch.randn(m, n, device="cuda", dtype=torch.float64)
    for layout in ("row", "col"):
        Al = A if layout == "row" else A.t().contiguous().t()
        for trans in (False, True):
            X = torch.randn(m if trans else n, l, device="cuda", dtype=torch.float64)
            for _ in range(2):
                sketch_product(Al, X, trans=trans)
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            torch.cuda.synchronize(); e0.record()
            for _ in range(5):
                sketch_product(Al, X, trans=trans)
            e1.record(); torch.cuda.synchronize()
            ms = e0.elapsed_time(e1) / 5
            gb = m * n * 8 / 1e9
            print(f"{m}x{n} l={l} {layout} trans={trans}: {ms:.3f} ms  {gb / ms * 1e3:.0f} GB/s  "
                  f"{2 * m * n * l / ms / 1e9:.1f} TF")
        del Al
