"""One config-2 decomposition (for ncu launch lists / captures).

    python scripts/profile_c2.py [--warm] [--n 32768] [--k 256 --p 32 --q 2]
"""
import argparse
import os
import sys
import warnings

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

ap = argparse.ArgumentParser()
ap.add_argument("--warm", action="store_true", help="run one untimed decomposition first")
ap.add_argument("--n", type=int, default=32768)
ap.add_argument("--k", type=int, default=256)
ap.add_argument("--p", type=int, default=32)
ap.add_argument("--q", type=int, default=2)
ap.add_argument("--dtype", default="float32")
args = ap.parse_args()

import torch  # noqa: E402

import bench  # noqa: E402
from paper_1706_07191_b200 import RankDeficiencyWarning, SketchConfig  # noqa: E402
from paper_1706_07191_b200.rsvd import run_rsvd  # noqa: E402

warnings.simplefilter("ignore", RankDeficiencyWarning)
bench.M = bench.N_COLS = args.n
A = bench.make_matrix(torch.device("cuda:0"))
if args.dtype == "float64":
    A = A.double()
cfg = SketchConfig(args.k, args.p, args.q)
if args.warm:
    run_rsvd(A, cfg, warn=False)
torch.cuda.synchronize()
r = run_rsvd(A, cfg, warn=False)
s = r.stats
print(f"wall {r.wall_seconds*1e3:.1f} ms  sketch {s.seconds_sketch*1e3:.1f}  orth "
      f"{s.seconds_orthonormalize*1e3:.1f}  core {s.seconds_form_core*1e3:.1f}  svd "
      f"{s.seconds_svd*1e3:.1f}  rank_y {s.detected_rank} rank_b {s.core_rank}")
