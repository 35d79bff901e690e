"""Where does the e2e (host-input) decomposition time go?  (GPU box probe)"""
import os, sys, time, warnings
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np
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
cfg = SketchConfig(256, 32, 2)
d = torch.empty_like(A)
for _ in range(2):
    torch.cuda.synchronize(); t0 = time.perf_counter()
    d.copy_(pinned, non_blocking=True); torch.cuda.synchronize()
    t = time.perf_counter() - t0
    print(f"raw H2D 4.29 GB: {t*1e3:.1f} ms = {A.numel()*4/t/1e9:.1f} GB/s")
for _ in range(3):
    t0 = time.perf_counter()
    r = run_rsvd(a_host, cfg, warn=False)
    t = time.perf_counter() - t0
    s = r.stats
    print(f"e2e {t*1e3:.1f} ms (C call {r.wall_seconds*1e3:.1f}): sketch {s.seconds_sketch*1e3:.1f} "
          f"orth {s.seconds_orthonormalize*1e3:.1f} core {s.seconds_form_core*1e3:.1f} svd {s.seconds_svd*1e3:.1f}")
t0 = time.perf_counter()
U = np.empty((32768, 288), dtype=np.float32, order="F"); Vt = np.empty((288, 32768), np.float32)
print(f"np.empty outputs {1e3*(time.perf_counter()-t0):.2f} ms")
x = torch.empty(32768 * 288, dtype=torch.float32, device=dev)
t0 = time.perf_counter(); x.cpu(); torch.cuda.synchronize()
print(f"D2H 37.7 MB pageable: {1e3*(time.perf_counter()-t0):.2f} ms")
