"""Scale sweep: rsvd_incore(s*A) vs rsvd_incore(A) for fp32/fp64 inputs."""
import numpy as np
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from oracle import ref_cpu
from paper_1706_07191_b200 import SketchConfig, rsvd_incore
import warnings
warnings.simplefilter("ignore")
for dt in (np.float32, np.float64):
    a = ref_cpu.lowrank_plus_noise(2048, 1536, 64, 1e-3, seed=4, dtype=dt)
    omega = ref_cpu.normal_sketch(1536, 80, 0, dtype=dt)
    for q in (0, 1, 2):
        f1 = rsvd_incore(a, SketchConfig(64, 16, q), omega=omega)
        for s in (1e-30, 1e-20, 1e-12, 1e-6, 1e6, 1e12, 1e30):
            try:
                fs = rsvd_incore((a.astype(np.float64) * s).astype(dt), SketchConfig(64, 16, q),
                                 omega=omega)
                err = np.max(np.abs(fs.sigma[:64] / s - f1.sigma[:64]) / f1.sigma[:64])
                print(f"{dt.__name__} q={q} s={s:g}: sigma rel err {err:.2e}")
            except Exception as e:
                print(f"{dt.__name__} q={q} s={s:g}: {type(e).__name__}")
