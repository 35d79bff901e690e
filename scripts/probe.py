"""GPU-box probes behind the numbers in DESIGN.md and profiles/ (one script,
one subcommand per probe; run under gpurun, results on stdout).

    python scripts/probe.py box        # host cores/RAM, pinned H2D/D2H, cuBLAS peaks
    python scripts/probe.py h2d        # pinned H2D with 1 / 2 / 4 concurrent streams
    python scripts/probe.py products   # config-2 tcgen05 products + fp64 C5/C1 products
    python scripts/probe.py e2e        # where the host-input (e2e) decomposition time goes
    python scripts/probe.py c1 [N]     # N config-1 decompositions (launch lists)
    python scripts/probe.py c5 [ITERS] # short config-5 RPCA run, per-iteration split
    python scripts/probe.py scale      # magnitude sweep s*A, in-core and streamed paths
    python scripts/probe.py sharded    # row-sharded driver at world size 1 vs single GPU
    python scripts/probe.py tcs [FLAGS...]  # product-kernel variants (BRSVD_TCS_FLAGS)
    python scripts/probe.py bias       # bias of tensor-core fp32 accumulation
    python scripts/probe.py lsweep     # config-2 product time against l
"""

import json
import os
import subprocess
import sys
import time
import warnings

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "scripts"))
warnings.simplefilter("ignore")


def _events():
    import torch
    return torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)


def _time(fn, reps=5, warm=2):
    import torch
    for _ in range(warm):
        fn()
    torch.cuda.synchronize()
    s, e = _events()
    s.record()
    for _ in range(reps):
        fn()
    e.record()
    torch.cuda.synchronize()
    return s.elapsed_time(e) / reps


def box(_):
    import torch
    out = {"cpu_count": os.cpu_count()}
    try:
        with open("/proc/meminfo") as f:
            out["mem_total_gb"] = int(f.readline().split()[1]) / 1e6
    except OSError:
        pass
    n = 1 << 28
    h = torch.empty(n, dtype=torch.float32, pin_memory=True).fill_(1.0)
    d = torch.empty(n, dtype=torch.float32, device="cuda")
    for name, fn in (("h2d", lambda: d.copy_(h, non_blocking=True)),
                     ("d2h", lambda: h.copy_(d, non_blocking=True))):
        out[f"pinned_{name}_gbs"] = n * 4 / (_time(fn) * 1e-3) / 1e9
    a = torch.randn(8192, 8192, device="cuda")
    b = torch.randn(8192, 8192, device="cuda")
    for name, tf32 in (("tf32", True), ("fp32_simt", False)):
        torch.backends.cuda.matmul.allow_tf32 = tf32
        out[f"cublas_{name}_tflops"] = 2 * 8192 ** 3 / (_time(lambda: a @ b) * 1e-3) / 1e12
    ad, bd = a.double(), b.double()
    out["cublas_fp64_tflops"] = 2 * 8192 ** 3 / (_time(lambda: ad @ bd, 2, 1) * 1e-3) / 1e12
    print(json.dumps(out))


def h2d(_):
    import torch
    n = 1 << 30
    h = torch.empty(n, dtype=torch.float32, pin_memory=True)
    d = torch.empty(n, dtype=torch.float32, device="cuda")
    for ns in (1, 2, 4):
        streams = [torch.cuda.Stream() for _ in range(ns)]
        for _ in range(2):
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            chunk = n // ns
            for i, s in enumerate(streams):
                with torch.cuda.stream(s):
                    d[i * chunk:(i + 1) * chunk].copy_(h[i * chunk:(i + 1) * chunk],
                                                       non_blocking=True)
            torch.cuda.synchronize()
            t = time.perf_counter() - t0
        print(f"{ns} stream(s): {n * 4 / t / 1e9:.1f} GB/s")


def products(_):
    import torch
    import bench
    from paper_1706_07191_b200.rsvd import sketch_product
    A = bench.make_matrix(torch.device("cuda:0"))
    X = torch.randn(288, 32768, device="cuda").t()
    for trans in (False, True):
        ms = _time(lambda: sketch_product(A, X, trans))
        print(f"config 2 trans={trans}: {ms:.3f} ms per product (incl. absmax + split)")
    del A, X
    torch.cuda.empty_cache()
    for (m, n, l) in [(76800, 20000, 20), (10000, 2000, 30)]:
        A = torch.randn(m, n, device="cuda", dtype=torch.float64)
        for layout in ("row", "col"):
            Al = A if layout == "row" else A.t().contiguous().t()
            for trans in (False, True):
                X = torch.randn(m if trans else n, l, device="cuda", dtype=torch.float64)
                ms = _time(lambda: sketch_product(Al, X, trans=trans))
                print(f"{m}x{n} fp64 l={l} {layout} trans={trans}: {ms:.3f} ms  "
                      f"{m * n * 8 / ms / 1e6:.0f} GB/s  {2 * m * n * l / ms / 1e9:.1f} TF")
            del Al
        del A
        torch.cuda.empty_cache()


def e2e(_):
    import numpy as np
    import torch
    import bench
    from paper_1706_07191_b200 import SketchConfig
    from paper_1706_07191_b200.rsvd import run_rsvd
    A = bench.make_matrix(torch.device("cuda:0"))
    pinned = torch.empty(A.shape, dtype=A.dtype, pin_memory=True)
    pinned.copy_(A)
    a_host = pinned.numpy()
    d = torch.empty_like(A)
    for _ in range(2):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        d.copy_(pinned, non_blocking=True)
        torch.cuda.synchronize()
        t = time.perf_counter() - t0
        print(f"raw H2D 4.29 GB: {t * 1e3:.1f} ms = {A.numel() * 4 / t / 1e9:.1f} GB/s")
    del d, A
    torch.cuda.empty_cache()
    cfg = SketchConfig(256, 32, 2)
    for _ in range(3):
        t0 = time.perf_counter()
        r = run_rsvd(a_host, cfg, warn=False)
        t = time.perf_counter() - t0
        s = r.stats
        print(f"e2e {t * 1e3:.1f} ms (C call {r.wall_seconds * 1e3:.1f}): sketch "
              f"{s.seconds_sketch * 1e3:.1f} orth {s.seconds_orthonormalize * 1e3:.1f} core "
              f"{s.seconds_form_core * 1e3:.1f} svd {s.seconds_svd * 1e3:.1f}")
    assert np.isfinite(r.factors.sigma).all()


def c1(argv):
    import numpy as np
    import torch
    from oracle import ref_cpu
    from paper_1706_07191_b200 import SketchConfig
    from paper_1706_07191_b200.rsvd import run_rsvd
    a = ref_cpu.lowrank_plus_noise(10000, 2000, 20, 1e-3, seed=1, dtype=np.float64)
    A = torch.from_numpy(a).cuda()
    cfg = SketchConfig(20, 10, 2)
    for _ in range(int(argv[0]) if argv else 5):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        run_rsvd(A, cfg, warn=False)
        torch.cuda.synchronize()
        print(f"{(time.perf_counter() - t0) * 1e3:.3f} ms")


def c5(argv):
    import torch
    from bench_configs import video_matrix
    from paper_1706_07191_b200 import RpcaConfig, ialm_rpca
    M = video_matrix(76800, 20000)
    iters = int(argv[0]) if argv else 3
    for _ in range(2):
        cfg = RpcaConfig(target_rank=10, oversampling=10, power_exponent=1, tol=1e-7,
                         max_iterations=iters)
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        res = ialm_rpca(M, cfg)
        torch.cuda.synchronize()
        print("iters", res.iterations, "total %.3f s" % (time.perf_counter() - t0),
              ["%.1f/%.1f" % (h["svd_seconds"] * 1e3, h["iter_seconds"] * 1e3)
               for h in res.history])


def scale(_):
    import numpy as np
    from oracle import ref_cpu
    from paper_1706_07191_b200 import SketchConfig, rsvd_incore
    from paper_1706_07191_b200.rsvd import run_rsvd, run_rsvd_stream
    for dt in (np.float32, np.float64):
        a = ref_cpu.lowrank_plus_noise(2048, 1536, 64, 1e-3, seed=4, dtype=dt)
        omega = ref_cpu.normal_sketch(1536, 80, 0, dtype=dt)
        for q in (0, 1, 2):
            f1 = rsvd_incore(a, SketchConfig(64, 16, q), omega=omega)
            for s in (1e-30, 1e-12, 1e-6, 1e6, 1e12, 1e30):
                try:
                    fs = rsvd_incore((a.astype(np.float64) * s).astype(dt),
                                     SketchConfig(64, 16, q), omega=omega)
                    err = np.max(np.abs(fs.sigma[:64] / s - f1.sigma[:64]) / f1.sigma[:64])
                    print(f"in-core {dt.__name__} q={q} s={s:g}: sigma rel err {err:.2e}")
                except Exception as e:
                    print(f"in-core {dt.__name__} q={q} s={s:g}: {type(e).__name__}")
    a = ref_cpu.lowrank_plus_noise(3000, 1200, 20, 1e-3, seed=21, dtype=np.float32)
    omega = ref_cpu.normal_sketch(1200, 30, 0, dtype=np.float32)
    cfg = SketchConfig(20, 10, 2)
    for order in ("C", "F"):
        ao = np.asarray(a, order=order)
        base = run_rsvd(ao, cfg, omega=omega, warn=False).factors.sigma[:20]
        for s in (1e-30, 1e-20, 1e-12, 1.0):
            try:
                st = run_rsvd_stream(np.asarray((a.astype(np.float64) * s).astype(np.float32),
                                                order=order), cfg, panel=257, nbuf=3,
                                     omega=omega, warn=False)
                print(f"streamed {order} s={s:g}",
                      np.max(np.abs(st.factors.sigma[:20] / s - base) / base))
            except Exception as e:
                print(f"streamed {order} s={s:g}", type(e).__name__, e)


def sharded(_):
    import torch
    import bench
    from paper_1706_07191_b200 import SketchConfig
    from paper_1706_07191_b200.distributed import GpuOps, TorchComm, rsvd_sharded
    from paper_1706_07191_b200.rsvd import run_rsvd
    A = bench.make_matrix(torch.device("cuda:0"))
    cfg = SketchConfig(256, 32, 2)
    comm, ops = TorchComm(), GpuOps(0)
    for name, fn in [("single", lambda: run_rsvd(A, cfg, warn=False).factors),
                     ("sharded w1", lambda: rsvd_sharded(A, cfg, 0, A.shape[0], comm=comm,
                                                         ops=ops)[0])]:
        for _ in range(3):
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            f = fn()
            torch.cuda.synchronize()
            t = time.perf_counter() - t0
        print(f"{name}: {t * 1e3:.1f} ms  sigma[:2] {[float(x) for x in f.sigma[:2]]}")


def tcs(argv):
    """Each BRSVD_TCS_FLAGS setting in a child process (profiles/r02_tcs_experiments.txt)."""
    if argv and argv[0] == "child":
        import torch
        from paper_1706_07191_b200.rsvd import sketch_product
        A = torch.randn(32768, 32768, device="cuda")
        X = torch.randn(32768, 288, device="cuda")
        for trans in (False, True):
            ms = _time(lambda: sketch_product(A, X, trans=trans))
            print(f"  flags={os.environ.get('BRSVD_TCS_FLAGS', '0')} "
                  f"tcs={os.environ.get('BRSVD_TCS', '1')} trans={trans}: {ms:.3f} ms")
        return
    for env in [{"BRSVD_TCS": "0"}] + [{"BRSVD_TCS_FLAGS": f} for f in (argv or ["0", "2"])]:
        e = dict(os.environ)
        e.update(env)
        subprocess.run([sys.executable, __file__, "tcs", "child"], env=e)


def lsweep(_):
    """Config-2 product time against the sketch width l (MMA N per CTA chunk):
    separates the per-MMA fixed cost from the N-proportional one."""
    import torch
    import bench
    from paper_1706_07191_b200.rsvd import sketch_product
    A = bench.make_matrix(torch.device("cuda:0"))
    for l in (16, 32, 64, 96, 128, 160, 192, 256, 288, 320):
        X = torch.randn(l, 32768, device="cuda").t()
        ms = _time(lambda: sketch_product(A, X, False))
        print(f"l={l:4d}: {ms:.3f} ms  {2 * 32768 ** 2 * l / ms / 1e9:.1f} TF/s")


def bias(_):
    import torch
    from paper_1706_07191_b200.rsvd import sketch_product
    torch.manual_seed(0)
    for K in (256, 2048, 16384):
        A = torch.rand(1024, K, device="cuda")
        X = torch.rand(K, 32, device="cuda")
        ref = A.double() @ X.double()
        rel = (sketch_product(A, X).double() - ref) / ref
        print(f"K={K:6d}  tensor-core product mean {rel.mean().item():+.3e} "
              f"max {rel.abs().max().item():.3e}")


if __name__ == "__main__":
    cmds = {f.__name__: f for f in (box, h2d, products, e2e, c1, c5, scale, sharded, tcs, bias, lsweep)}
    if len(sys.argv) < 2 or sys.argv[1] not in cmds:
        print(__doc__)
        sys.exit(2)
    cmds[sys.argv[1]](sys.argv[2:])
