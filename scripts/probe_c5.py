"""Short C5 RPCA run (3 iterations) for launch lists."""
import os, sys, time
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "scripts"))
import torch
from bench_configs import video_matrix
from paper_1706_07191_b200 import RpcaConfig, ialm_rpca
M = video_matrix(76800, 20000)
cfg = RpcaConfig(target_rank=10, oversampling=10, power_exponent=1, tol=1e-7, max_iterations=int(sys.argv[1]) if len(sys.argv) > 1 else 3)
torch.cuda.synchronize(); t0 = time.perf_counter()
res = ialm_rpca(M, cfg)
torch.cuda.synchronize()
print("iters", res.iterations, "total %.3f s" % (time.perf_counter() - t0),
      ["%.1f/%.1f" % (h["svd_seconds"] * 1e3, h["iter_seconds"] * 1e3) for h in res.history])
