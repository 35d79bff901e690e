"""Time the row-sharded driver at world size 1 against the single-GPU pipeline."""
import os, sys, time, warnings
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch
import bench
from paper_1706_07191_b200 import SketchConfig, RankDeficiencyWarning
from paper_1706_07191_b200.rsvd import run_rsvd
from paper_1706_07191_b200.distributed import GpuOps, TorchComm, rsvd_sharded
warnings.simplefilter("ignore", RankDeficiencyWarning)
dev = torch.device("cuda:0")
A = bench.make_matrix(dev)
cfg = SketchConfig(256, 32, 2)
comm, ops = TorchComm(), GpuOps(0)
for name, fn in [("single", lambda: run_rsvd(A, cfg, warn=False).factors),
                 ("sharded w1", lambda: rsvd_sharded(A, cfg, 0, A.shape[0], comm=comm, ops=ops)[0])]:
    for i in range(3):
        torch.cuda.synchronize(); t0 = time.perf_counter()
        f = fn()
        torch.cuda.synchronize()
        t = time.perf_counter() - t0
    print(f"{name}: {t*1e3:.1f} ms  sigma[:2] {f.sigma[:2].tolist() if hasattr(f.sigma,'tolist') else f.sigma[:2]}")
