"""Magnitude sweep of the streamed (out-of-core) path, fp32."""
import os, sys, warnings
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
from oracle import ref_cpu
from paper_1706_07191_b200 import SketchConfig
from paper_1706_07191_b200.rsvd import run_rsvd, run_rsvd_stream
warnings.simplefilter("ignore")
a = ref_cpu.lowrank_plus_noise(3000, 1200, 20, 1e-3, seed=21, dtype=np.float32)
omega = ref_cpu.normal_sketch(1200, 30, 0, dtype=np.float32)
cfg = SketchConfig(20, 10, 2)
base = run_rsvd(a, cfg, omega=omega, warn=False).factors.sigma[:20]
for s in (1e-30, 1e-20, 1e-12, 1.0):
    try:
        st = run_rsvd_stream((a.astype(np.float64) * s).astype(np.float32), cfg, panel=257,
                             nbuf=3, omega=omega, warn=False)
        print(s, np.max(np.abs(st.factors.sigma[:20] / s - base) / base))
    except Exception as e:
        print(s, type(e).__name__, e)
# column-major input: the column-panel path
ac = np.asfortranarray(a)
base = run_rsvd(ac, cfg, omega=omega, warn=False).factors.sigma[:20]
for s in (1e-30, 1e-20, 1e-12, 1.0):
    try:
        st = run_rsvd_stream(np.asfortranarray((a.astype(np.float64) * s).astype(np.float32)),
                             cfg, panel=257, nbuf=3, omega=omega, warn=False)
        print("col", s, np.max(np.abs(st.factors.sigma[:20] / s - base) / base))
    except Exception as e:
        print("col", s, type(e).__name__, e)
