"""Measure the bias of tensor-core fp32 accumulation (3xTF32 product) on
coherent sums: positive A and X, compare with the fp64 product."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_1706_07191_b200.rsvd import sketch_product
torch.manual_seed(0)
for K in (256, 2048, 16384):
    A = torch.rand(1024, K, device="cuda")
    X = torch.rand(K, 32, device="cuda")
    C = sketch_product(A, X).double()
    ref = A.double() @ X.double()
    rel = (C - ref) / ref
    Cf = (A @ X).double() if False else None
    torch.backends.cuda.matmul.allow_tf32 = False
    Ct = (A @ X).double()
    relt = (Ct - ref) / ref
    print(f"K={K:6d}  tc3xtf32 mean {rel.mean().item():+.3e} max {rel.abs().max().item():.3e} | "
          f"cublas fp32 mean {relt.mean().item():+.3e} max {relt.abs().max().item():.3e}")
