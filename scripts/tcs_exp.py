"""Product-kernel experiment timing: one K-major and one MN-major config-2
product per BRSVD_TCS_FLAGS setting (CUDA events; results ignored)."""
import os, sys, subprocess
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
if len(sys.argv) > 1 and sys.argv[1] == "child":
    import torch
    from paper_1706_07191_b200.rsvd import sketch_product
    A = torch.randn(32768, 32768, device="cuda")
    X = torch.randn(32768, 288, device="cuda")
    for trans in (False, True):
        for _ in range(2):
            sketch_product(A, X, trans=trans)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(5):
            sketch_product(A, X, trans=trans)
        e1.record()
        torch.cuda.synchronize()
        print(f"  flags={os.environ.get('BRSVD_TCS_FLAGS','0')} tcs={os.environ.get('BRSVD_TCS','1')} trans={trans}: {e0.elapsed_time(e1)/5:.3f} ms")
    sys.exit(0)
FL = sys.argv[1:] if len(sys.argv) > 1 else ["0", "2", "4", "6"]
for env in [{"BRSVD_TCS": "0"}] + [{"BRSVD_TCS_FLAGS": f} for f in FL]:
    e = dict(os.environ); e.update(env)
    subprocess.run([sys.executable, __file__, "child"], env=e)
