import os, sys, torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1706_07191_b200.rsvd import sketch_product
m, n, l = 76800, 20000, 20
A = torch.randn(m, n, device="cuda", dtype=torch.float64)
trans = len(sys.argv) > 1 and sys.argv[1] == "t"
X = torch.randn(m if trans else n, l, device="cuda", dtype=torch.float64)
for _ in range(2):
    sketch_product(A, X, trans=trans)
torch.cuda.synchronize()
