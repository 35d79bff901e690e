import numpy as np, os, sys, warnings
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from oracle import ref_cpu
from paper_1706_07191_b200 import SketchConfig, rsvd_incore
warnings.simplefilter("ignore")
a = ref_cpu.lowrank_plus_noise(2048, 1536, 64, 1e-3, seed=4, dtype=np.float32)
print("max|a|", np.abs(a).max())
omega = ref_cpu.normal_sketch(1536, 80, 0, dtype=np.float32)
f1 = rsvd_incore(a, SketchConfig(64, 16, 1), omega=omega)
print("ref", f1.sigma[:4])
for s in (1e-20, 1e-30):
    try:
        fs = rsvd_incore((a.astype(np.float64) * s).astype(np.float32), SketchConfig(64, 16, 1), omega=omega)
        print(s, fs.sigma[:4] / s, fs.sigma[60:64] / s)
    except Exception as e:
        print(s, repr(e))
