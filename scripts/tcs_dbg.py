import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_1706_07191_b200.rsvd import sketch_product
A = torch.randn(32768, 32768, device="cuda")
X = torch.randn(32768, 288, device="cuda")
sketch_product(A, X)
torch.cuda.synchronize()
os.environ["BRSVD_TCS_DEBUG"] = "1"
sketch_product(A, X)
