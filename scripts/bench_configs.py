"""Bench lines for the other BASELINE configurations (not the driver's
headline, which is bench.py / config 2).  One JSON line per config.

    python scripts/bench_configs.py [--configs c1,c3,c5] [--c3-rows 100000]

  c1  in-core fp64 10000x2000 rank-20 + 1e-3 noise, k=20 p=10 q=2 (device A)
  c3  out-of-core fp32 rows x 100000 rank-100 + noise, k=100 p=20 q=1, A in
      pinned host memory streamed over PCIe (the full 1e6 rows = 400 GB exceed
      this box's 196 GB of host RAM; the default is the 1/10 row sample the
      survey's CPU plan uses, 40 GB).  Roofline: measured pinned H2D.
  c4  the c3 matrix row-sharded over torchrun ranks, one host-resident pinned
      shard per GPU streamed over its own link (distributed.HostShard), NCCL
      all-reduce of Z / Grams / B^T; roofline: concurrent pinned H2D.
      torchrun --nproc-per-node N scripts/bench_configs.py --configs c4
  c5  IALM-RPCA fp64 76800 x 20000 (12.3 GB, in HBM), low-rank background +
      moving sparse foreground, k=p=10, q=1, tol 1e-7 (ialm_rpca).
"""

import argparse
import json
import os
import sys
import time
import warnings

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def pinned_h2d_gbs():
    import torch
    n = 1 << 28
    h = torch.empty(n, dtype=torch.float32, pin_memory=True)
    d = torch.empty(n, dtype=torch.float32, device="cuda")
    d.copy_(h)
    torch.cuda.synchronize()
    best = 1e9
    for _ in range(3):
        s, e = torch.cuda.Event(True), torch.cuda.Event(True)
        s.record()
        d.copy_(h, non_blocking=True)
        e.record()
        torch.cuda.synchronize()
        best = min(best, s.elapsed_time(e) / 1e3)
    return n * 4 / best / 1e9


def bench_c1(steps):
    import torch
    from oracle import ref_cpu
    from paper_1706_07191_b200 import SketchConfig
    from paper_1706_07191_b200.rsvd import run_rsvd
    a = ref_cpu.lowrank_plus_noise(10000, 2000, 20, 1e-3, seed=1)
    A = torch.as_tensor(a, device="cuda")
    cfg = SketchConfig(20, 10, 2)
    for _ in range(3):
        run_rsvd(A, cfg, warn=False)
    torch.cuda.synchronize()
    s, e = torch.cuda.Event(True), torch.cuda.Event(True)
    s.record()
    for _ in range(steps):
        run_rsvd(A, cfg, warn=False)
    e.record()
    torch.cuda.synchronize()
    t = s.elapsed_time(e) / 1e3 / steps
    t0 = time.perf_counter()
    ref_cpu.randomized_svd(a, 20, 10, 2, seed=0)
    tc = time.perf_counter() - t0
    passes = 4
    return {"config": "c1", "seconds": t, "a_stream_gbs": passes * a.nbytes / t / 1e9,
            "cpu_seconds": tc, "cpu_cores": os.cpu_count(), "speedup_vs_cpu": tc / t,
            "m": 10000, "n": 2000, "dtype": "f64", "k": 20, "p": 10, "q": 2}


def bench_c3(rows, steps):
    import torch
    from paper_1706_07191_b200 import SketchConfig
    from paper_1706_07191_b200.rsvd import run_rsvd_stream
    n, rank = 100000, 100
    host = torch.empty((rows, n), dtype=torch.float32, pin_memory=True)
    g = torch.Generator(device="cuda").manual_seed(5)
    R = torch.randn(rank, n, generator=g, device="cuda")
    chunk = 8192
    for r0 in range(0, rows, chunk):
        r1 = min(rows, r0 + chunk)
        L = torch.randn(r1 - r0, rank, generator=g, device="cuda")
        blk = L @ R
        blk.add_(torch.randn(r1 - r0, n, generator=g, device="cuda"), alpha=1e-3)
        host[r0:r1].copy_(blk)
    del R, L, blk
    torch.cuda.synchronize()
    torch.cuda.empty_cache()
    a = host.numpy()
    cfg = SketchConfig(100, 20, 1)
    panel = 8192
    run_rsvd_stream(a, cfg, panel=panel, nbuf=3, warn=False)   # warm-up
    ts = []
    for _ in range(steps):
        t0 = time.perf_counter()
        run = run_rsvd_stream(a, cfg, panel=panel, nbuf=3, warn=False)
        ts.append(time.perf_counter() - t0)
    t = float(np.median(ts))
    passes = run.stats.words_read // (rows * n)
    gbs = passes * rows * n * 4 / t / 1e9
    peak = pinned_h2d_gbs()
    return {"config": "c3_rows_sample", "rows": rows, "n": n, "dtype": "f32", "k": 100,
            "p": 20, "q": 1, "host_bytes": rows * n * 4, "passes": int(passes),
            "seconds": t, "a_stream_gbs": gbs,
            "roofline": {"bound": "pcie_h2d", "achieved": gbs, "peak": peak, "unit": "GB/s",
                         "frac": gbs / peak, "peak_basis": "measured pinned H2D, 1 GiB"},
            "panel_rows": panel, "nbuf": 3,
            "stages_s": {"sketch+power": run.stats.seconds_sketch,
                         "orthonormalize": run.stats.seconds_orthonormalize,
                         "form_core": run.stats.seconds_form_core,
                         "svd": run.stats.seconds_svd}}


def _dist():
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    import torch
    torch.cuda.set_device(local % max(1, torch.cuda.device_count()))
    if world > 1:
        import torch.distributed as dist
        os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
        if not dist.is_initialized():
            dist.init_process_group("nccl", device_id=torch.device(
                f"cuda:{local % max(1, torch.cuda.device_count())}"))
    return world, rank, local


def _max_over_ranks(x, world):
    if world == 1:
        return x
    import torch
    import torch.distributed as dist
    t = torch.tensor([x], dtype=torch.float64, device="cuda")
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def _barrier(world):
    if world > 1:
        import torch.distributed as dist
        dist.barrier()


def concurrent_h2d_gbs(world):
    """Aggregate pinned H2D with every rank copying 1 GiB at once (the C4
    roofline denominator: host memory and the PCIe links all busy)."""
    import torch
    n = 1 << 28
    h = torch.empty(n, dtype=torch.float32, pin_memory=True)
    d = torch.empty(n, dtype=torch.float32, device="cuda")
    d.copy_(h)
    torch.cuda.synchronize()
    best = 1e9
    for _ in range(3):
        _barrier(world)
        s, e = torch.cuda.Event(True), torch.cuda.Event(True)
        s.record()
        d.copy_(h, non_blocking=True)
        e.record()
        torch.cuda.synchronize()
        best = min(best, _max_over_ranks(s.elapsed_time(e) / 1e3, world))
    return world * n * 4 / best / 1e9


def bench_c4(rows_total, steps):
    """Config 4 structure: the (rows_total x 1e5) fp32 rank-100 + noise matrix
    row-sharded over the ranks, each shard host-resident in pinned memory and
    streamed over its own PCIe link (distributed.HostShard), Z / Gram / B^T
    all-reduced over NCCL.  Strong scaling over the fixed matrix."""
    import torch
    from paper_1706_07191_b200 import SketchConfig
    from paper_1706_07191_b200.distributed import GpuOps, HostShard, TorchComm, rsvd_sharded
    world, rank, local = _dist()
    n, rk = 100000, 100
    bounds = np.linspace(0, rows_total, world + 1).astype(np.int64)
    r0, r1 = int(bounds[rank]), int(bounds[rank + 1])
    host = torch.empty((r1 - r0, n), dtype=torch.float32, pin_memory=True)
    gR = torch.Generator(device="cuda").manual_seed(5)          # shared right factor
    R = torch.randn(rk, n, generator=gR, device="cuda")
    g = torch.Generator(device="cuda").manual_seed(1000 + rank)
    chunk = 8192
    for c0 in range(0, r1 - r0, chunk):
        c1 = min(r1 - r0, c0 + chunk)
        blk = torch.randn(c1 - c0, rk, generator=g, device="cuda") @ R
        blk.add_(torch.randn(c1 - c0, n, generator=g, device="cuda"), alpha=1e-3)
        host[c0:c1].copy_(blk)
    del R, blk
    torch.cuda.synchronize()
    torch.cuda.empty_cache()
    shard = HostShard(host.numpy(), panel=8192, nbuf=3)
    cfg = SketchConfig(100, 20, 1)
    comm, ops = TorchComm(), GpuOps()
    rsvd_sharded(shard, cfg, r0, rows_total, comm=comm, ops=ops)   # warm-up
    ts = []
    for _ in range(steps):
        shard.passes, shard.pass_ms = 0, []
        _barrier(world)
        torch.cuda.synchronize()
        s, e = torch.cuda.Event(True), torch.cuda.Event(True)
        s.record()
        f, info = rsvd_sharded(shard, cfg, r0, rows_total, comm=comm, ops=ops)
        e.record()
        torch.cuda.synchronize()
        ts.append(_max_over_ranks(s.elapsed_time(e) / 1e3, world))
    t = float(np.median(ts))
    passes = info["passes"]
    gbs = passes * rows_total * n * 4 / t / 1e9
    peak = concurrent_h2d_gbs(world)
    return {"config": "c4_rowshard_stream", "gpus": world, "rows": rows_total, "n": n,
            "dtype": "f32", "k": 100, "p": 20, "q": 1, "host_bytes": rows_total * n * 4,
            "passes": passes, "seconds": t, "a_stream_gbs": gbs, "scaling": "strong",
            "roofline": {"bound": "pcie_h2d", "achieved": gbs, "peak": peak, "unit": "GB/s",
                         "frac": gbs / peak,
                         "peak_basis": f"measured concurrent pinned H2D, {world} GPU(s)"},
            "sigma_top3": [float(x) for x in f.sigma[:3].cpu()], "rank": rank}


def video_matrix(m, n, seed=0):
    """Low-rank nonnegative background (rank 3) + moving blocks."""
    import torch
    g = torch.Generator(device="cuda").manual_seed(seed)
    Lb = torch.rand(m, 3, generator=g, device="cuda", dtype=torch.float64)
    Rb = torch.rand(3, n, generator=g, device="cuda", dtype=torch.float64)
    M = Lb @ Rb
    side = 240                                         # frame 320 x 240 = 76800
    j = torch.arange(n, device="cuda")
    x0 = (j * 3) % (320 - 16)                          # moving 16 x 16 block
    d = torch.arange(16, device="cuda")
    idx = ((x0[:, None, None] + d[None, :, None]) * side + 100 + d[None, None, :])
    M[idx.reshape(n, -1), j[:, None]] = 1.0
    return M


def bench_c5(steps):
    import torch
    from oracle import ref_cpu
    from paper_1706_07191_b200 import RpcaConfig, ialm_rpca
    M = video_matrix(76800, 20000)
    cfg = RpcaConfig(target_rank=10, oversampling=10, power_exponent=1, tol=1e-7)
    # warm-up at full size (module load + the device pool's first growth)
    ialm_rpca(M, RpcaConfig(target_rank=10, oversampling=10, power_exponent=1, tol=1e-7,
                            max_iterations=1))
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    res = ialm_rpca(M, cfg)
    torch.cuda.synchronize()
    t = time.perf_counter() - t0
    # CPU reference on the 1/10 column slice (~3.7 min on 8 cores)
    Ms = M[:, :2000].cpu().numpy()
    t1 = time.perf_counter()
    ref = ref_cpu.ialm(Ms, 10, 10, 1, tol=1e-7, max_iterations=5)
    tcpu5 = time.perf_counter() - t1
    per_it_cpu_slice = tcpu5 / max(ref["iterations"], 1)
    return {"config": "c5", "m": 76800, "n": 20000, "dtype": "f64", "seconds": t,
            "iterations": res.iterations, "converged": res.converged,
            "seconds_per_iteration": t / max(res.iterations, 1),
            "svd_seconds_total": sum(h["svd_seconds"] for h in res.history),
            "cpu_seconds_per_iteration_on_1_10_slice": per_it_cpu_slice,
            "cpu_seconds_per_iteration_full_est": per_it_cpu_slice * 10,
            "cpu_cores": os.cpu_count()}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--configs", default="c1,c3,c5")
    ap.add_argument("--c3-rows", type=int, default=100000)
    ap.add_argument("--steps", type=int, default=3)
    args = ap.parse_args()
    from paper_1706_07191_b200 import RankDeficiencyWarning
    warnings.simplefilter("ignore", RankDeficiencyWarning)
    for c in args.configs.split(","):
        if c == "c1":
            out = bench_c1(max(args.steps, 10))
        elif c == "c3":
            out = bench_c3(args.c3_rows, args.steps)
        elif c == "c5":
            out = bench_c5(args.steps)
        elif c == "c4":
            out = bench_c4(args.c3_rows, args.steps)
            if out.pop("rank") != 0:
                continue
        else:
            continue
        print(json.dumps(out), flush=True)


if __name__ == "__main__":
    main()
