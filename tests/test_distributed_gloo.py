"""Row-sharded driver (config 4 logic) over world_size-2 gloo on CPU.

The stage operations are numpy (tests/dist_numpy_ops.py); what is tested is
the sharding, the collectives and the replicated steps of
paper_1706_07191_b200.distributed.rsvd_sharded against the single-process
oracle (global power iteration, oracle/ref_cpu.py).
"""

import os
import socket

import numpy as np
import pytest


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, case, out_dir, streamed=False):
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    sys.path.insert(0, root)
    import torch.distributed as dist
    from paper_1706_07191_b200 import SketchConfig
    from paper_1706_07191_b200.distributed import TorchComm, rsvd_sharded
    from tests.dist_numpy_ops import NumpyOps
    dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port}", rank=rank,
                            world_size=world)
    A, cfg_args = _case(case)
    m = A.shape[0]
    bounds = np.linspace(0, m, world + 1).astype(int)
    r0, r1 = bounds[rank], bounds[rank + 1]
    shard = A[r0:r1].copy()
    if streamed:   # host-resident shard streamed in row panels (config 4)
        from paper_1706_07191_b200.distributed import HostShard
        shard = HostShard(shard if case != "f32" else np.asfortranarray(shard), panel=37)
    f, info = rsvd_sharded(shard, SketchConfig(**cfg_args), r0, m,
                           comm=TorchComm(), ops=NumpyOps())
    if streamed:
        assert info["passes"] == cfg_args["power_exponent"] + 2
    np.savez(os.path.join(out_dir, f"r{rank}.npz"), U=f.U, sigma=f.sigma, Vt=f.Vt, r0=r0,
             rank_y=info["rank_y"], rank_b=info["rank_b"])
    dist.barrier()
    dist.destroy_process_group()


def _case(name):
    from oracle import ref_cpu
    if name == "noisy":
        return (ref_cpu.lowrank_plus_noise(600, 300, 10, 1e-3, seed=3),
                dict(target_rank=10, oversampling=6, power_exponent=2, master_seed=5))
    if name == "deficient":
        return (ref_cpu.lowrank_plus_noise(400, 200, 5, 0.0, seed=4),
                dict(target_rank=5, oversampling=11, power_exponent=1, master_seed=1))
    if name == "f32":
        return (ref_cpu.lowrank_plus_noise(512, 256, 12, 1e-3, seed=5, dtype=np.float32),
                dict(target_rank=12, oversampling=8, power_exponent=1, master_seed=2))
    raise KeyError(name)


def _run(case, world, tmp_path, streamed=False):
    import torch.multiprocessing as mp
    port = _free_port()
    mp.start_processes(_worker, args=(world, port, case, str(tmp_path), streamed),
                       nprocs=world, join=True, start_method="spawn")
    parts = [np.load(tmp_path / f"r{r}.npz") for r in range(world)]
    U = np.vstack([p["U"] for p in parts])
    return U, parts


@pytest.mark.parametrize("streamed", [False, True])
@pytest.mark.parametrize("case", ["noisy", "f32"])
def test_sharded_matches_single_process_oracle(case, streamed, tmp_path):
    """In-memory shards and host-resident shards streamed in row panels
    (q + 2 passes, fp64 Z accumulation) against the single-process oracle."""
    from oracle import ref_cpu
    U, parts = _run(case, 2, tmp_path, streamed)
    A, cfg = _case(case)
    k, p, q, seed = (cfg["target_rank"], cfg["oversampling"], cfg["power_exponent"],
                     cfg["master_seed"])
    ref = ref_cpu.randomized_svd(A, k, p, q, seed)
    fp64 = A.dtype == np.float64
    for part in parts:   # sigma and Vt are replicated and identical
        np.testing.assert_array_equal(part["sigma"], parts[0]["sigma"])
        np.testing.assert_array_equal(part["Vt"], parts[0]["Vt"])
    np.testing.assert_allclose(parts[0]["sigma"][:k], ref["sigma"][:k],
                               rtol=1e-10 if fp64 else 1e-5)
    np.testing.assert_allclose(U[:, :k], ref["U"][:, :k], atol=1e-8 if fp64 else 2e-3)
    np.testing.assert_allclose(parts[0]["Vt"][:k], ref["Vt"][:k], atol=1e-8 if fp64 else 2e-3)


def test_sharded_rank_deficient_completion(tmp_path):
    U, parts = _run("deficient", 2, tmp_path)
    l = U.shape[1]
    assert np.linalg.norm(U.T @ U - np.eye(l)) <= 100 * l * np.finfo(np.float64).eps
    assert int(parts[0]["rank_y"]) == 5
    Vt = parts[0]["Vt"]
    assert np.linalg.norm(Vt @ Vt.T - np.eye(l)) <= 100 * l * np.finfo(np.float64).eps
    s = parts[0]["sigma"]
    assert s[5] <= 1e-10 * s[0]


def _guard_worker(rank, world, port, frac, q, out_dir):
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    sys.path.insert(0, root)
    import torch.distributed as dist
    from oracle import ref_cpu
    from paper_1706_07191_b200 import SketchConfig
    from paper_1706_07191_b200.distributed import TorchComm, rsvd_sharded
    from tests.dist_numpy_ops import NumpyOps
    dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port}", rank=rank,
                            world_size=world)
    a = ref_cpu.lowrank_plus_noise(300, 200, 5, 1e-2, seed=8)
    omega = ref_cpu.normal_sketch(200, 10, 0, dtype=np.float64)
    peak1 = float(np.max(np.abs(ref_cpu.power_sample(a, omega, q))))
    c = (frac * 0.01 * float(np.finfo(np.float64).max) / peak1) ** (1.0 / (2 * q + 1))
    ac = a * c
    r0, r1 = (0, 140) if rank == 0 else (140, 300)
    fired = False
    try:
        rsvd_sharded(ac[r0:r1].copy(), SketchConfig(5, 5, q), r0, 300, comm=TorchComm(),
                     ops=NumpyOps(), omega=omega)
    except FloatingPointError:
        fired = True
    np.save(os.path.join(out_dir, f"g{rank}.npy"), np.array([fired]))
    dist.destroy_process_group()


@pytest.mark.parametrize("q", [1, 2])
@pytest.mark.parametrize("frac", [0.99, 1.01])
def test_sharded_overflow_guard_is_exact(frac, q, tmp_path):
    """_check_overflow (rsvd.py:84-91) in the row-sharded driver: inputs that
    put the reference's unnormalised sample at 0.99x / 1.01x of 0.01 *
    finfo.max fire exactly when the reference does, on every rank (the peak
    is formed from each rank's rows and the kept basis changes, then
    all-reduced)."""
    import torch.multiprocessing as mp
    mp.start_processes(_guard_worker, args=(2, _free_port(), frac, q, str(tmp_path)),
                       nprocs=2, join=True, start_method="spawn")
    fired = [bool(np.load(tmp_path / f"g{r}.npy")[0]) for r in range(2)]
    assert fired == [frac > 1.0] * 2
