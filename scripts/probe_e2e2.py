"""bench-style e2e loop: per-call wall vs C-call time."""
import os, sys, time, warnings
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch
import bench
from paper_1706_07191_b200 import SketchConfig, RankDeficiencyWarning
from paper_1706_07191_b200.rsvd import run_rsvd
warnings.simplefilter("ignore", RankDeficiencyWarning)
dev = torch.device("cuda:0")
A = bench.make_matrix(dev)
pinned = torch.empty(A.shape, dtype=A.dtype, pin_memory=True)
pinned.copy_(A)
a_host = pinned.numpy()
del A
torch.cuda.empty_cache()
cfg = SketchConfig(256, 32, 2)
out = None
for i in range(8):
    t0 = time.perf_counter()
    r = run_rsvd(a_host, cfg, warn=False)
    out = (r.factors.U, r.factors.sigma, r.factors.Vt)
    float(out[1][0])
    t = time.perf_counter() - t0
    print(f"call {i}: {t*1e3:.1f} ms, C call {r.wall_seconds*1e3:.1f} ms")
