"""C1 (fp64 10000x2000, k=20 p=10 q=2) decompositions for launch lists."""
import os, sys, time, warnings
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np, torch
from oracle import ref_cpu
from paper_1706_07191_b200 import SketchConfig, RankDeficiencyWarning
from paper_1706_07191_b200.rsvd import run_rsvd
warnings.simplefilter("ignore", RankDeficiencyWarning)
a = ref_cpu.lowrank_plus_noise(10000, 2000, 20, 1e-3, seed=1, dtype=np.float64)
A = torch.from_numpy(a).cuda()
cfg = SketchConfig(20, 10, 2)
for i in range(int(sys.argv[1]) if len(sys.argv) > 1 else 5):
    torch.cuda.synchronize(); t0 = time.perf_counter()
    r = run_rsvd(A, cfg, warn=False)
    torch.cuda.synchronize()
    print(f"{(time.perf_counter() - t0) * 1e3:.3f} ms")
