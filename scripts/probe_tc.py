"""Time one config-2 A-streaming product (device A) -- kernel experiments."""
import os, sys, time
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch
import bench
from paper_1706_07191_b200.rsvd import sketch_product
A = bench.make_matrix(torch.device("cuda:0"))
X = torch.randn(288, 32768, device="cuda").t()
for trans in (False, True):
    for _ in range(2):
        sketch_product(A, X, trans)
    torch.cuda.synchronize()
    s, e = torch.cuda.Event(True), torch.cuda.Event(True)
    s.record()
    for _ in range(5):
        sketch_product(A, X, trans)
    e.record(); torch.cuda.synchronize()
    print(f"trans={trans}: {s.elapsed_time(e)/5:.3f} ms per product (incl. absmax + split)")
