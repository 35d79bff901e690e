"""C5 RPCA: per-call wall time split (repeat in one process)."""
import os, sys, time
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "scripts"))
import torch
from bench_configs import video_matrix
from paper_1706_07191_b200 import RpcaConfig, ialm_rpca
M = video_matrix(76800, 20000)
for rep in range(3):
    cfg = RpcaConfig(target_rank=10, oversampling=10, power_exponent=1, tol=1e-7, max_iterations=3)
    torch.cuda.synchronize(); t0 = time.perf_counter()
    res = ialm_rpca(M, cfg)
    torch.cuda.synchronize()
    print("iters", res.iterations, "total %.3f s" % (time.perf_counter() - t0),
          "sum iter %.3f" % sum(h["iter_seconds"] for h in res.history))
