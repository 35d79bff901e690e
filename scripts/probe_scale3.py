import numpy as np, os, sys, warnings, torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from oracle import ref_cpu
from paper_1706_07191_b200.rsvd import sketch_product
from paper_1706_07191_b200.distributed import GpuOps
ops = GpuOps()
a = ref_cpu.lowrank_plus_noise(2048, 1536, 64, 1e-3, seed=4, dtype=np.float32)
omega = ref_cpu.normal_sketch(1536, 80, 0, dtype=np.float32)
for s in (1.0, 1e-20):
    A = torch.tensor((a.astype(np.float64) * s).astype(np.float32), device="cuda")
    X = torch.tensor(omega, device="cuda")
    Y = sketch_product(A, X)
    Z = sketch_product(A, Y * (1 / Y.abs().max()), trans=True).contiguous().t().contiguous().t()
    print(s, "Z max", Z.abs().max().item())
    G = ops.gram(Z)
    print(s, "G diag", torch.as_tensor(G).diagonal()[:3])
    Zn = ops.normalize(Z)
    Zn = torch.as_tensor(Zn)
    print(s, "Zn finite", torch.isfinite(Zn).all().item(), Zn.abs().max().item(),
          (Zn.double().t() @ Zn.double()).diagonal()[:3])
