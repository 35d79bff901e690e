"""Row-sharded driver on the GPU: two ranks sharing cuda:0 over gloo (the
box has one GPU), GPU stage operations through the C ABI, against the
single-GPU pipeline with the same sketch."""

import os
import socket

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, dtype_name, out_dir, streamed=False):
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    sys.path.insert(0, root)
    import torch
    import torch.distributed as dist
    from oracle import ref_cpu
    from paper_1706_07191_b200 import RankDeficiencyWarning, SketchConfig
    from paper_1706_07191_b200.distributed import GpuOps, TorchComm, rsvd_sharded
    import warnings
    warnings.simplefilter("ignore", RankDeficiencyWarning)
    torch.cuda.set_device(0)
    dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port}", rank=rank,
                            world_size=world)
    dtype = np.float64 if dtype_name == "f64" else np.float32
    A = ref_cpu.lowrank_plus_noise(3000, 800, 20, 1e-3, seed=9, dtype=dtype)
    omega = ref_cpu.normal_sketch(800, 30, 0, dtype=dtype)
    bounds = [0, 1500, 3000]
    r0, r1 = bounds[rank], bounds[rank + 1]
    if streamed:
        # host-resident shard in pinned memory, streamed in 301-row panels
        # (the f32 case as a column-major shard: strided row panels)
        from paper_1706_07191_b200.distributed import HostShard
        pin = torch.empty(A[r0:r1].shape[::-1] if dtype_name == "f32" else A[r0:r1].shape,
                          dtype=torch.float64 if dtype == np.float64 else torch.float32,
                          pin_memory=True).numpy()
        host = pin.T if dtype_name == "f32" else pin
        host[...] = A[r0:r1]
        A_loc = HostShard(host, panel=301, nbuf=3)
    else:
        A_loc = torch.as_tensor(A[r0:r1], device="cuda")
    f, info = rsvd_sharded(A_loc, SketchConfig(20, 10, 2), r0, 3000, comm=TorchComm(),
                           ops=GpuOps(0), omega=omega)
    if streamed:
        assert info["passes"] == 4 and info["h2d_bytes"] == 4 * A[r0:r1].nbytes
    np.savez(os.path.join(out_dir, f"r{rank}.npz"), U=f.U.cpu().numpy(),
             sigma=f.sigma.cpu().numpy(), Vt=f.Vt.cpu().numpy())
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("streamed", [False, True])
@pytest.mark.parametrize("dtype_name", ["f64", "f32"])
def test_two_shards_match_single_gpu(dtype_name, streamed, tmp_path):
    """Resident shards and host-resident shards streamed through the panel
    streamer (config 4's path) against the single-GPU decomposition."""
    import torch.multiprocessing as mp
    from oracle import ref_cpu
    from paper_1706_07191_b200 import SketchConfig, rsvd_incore
    mp.start_processes(_worker, args=(2, _free_port(), dtype_name, str(tmp_path), streamed),
                       nprocs=2, join=True, start_method="spawn")
    parts = [np.load(tmp_path / f"r{r}.npz") for r in range(2)]
    U = np.vstack([p["U"] for p in parts])
    dtype = np.float64 if dtype_name == "f64" else np.float32
    A = ref_cpu.lowrank_plus_noise(3000, 800, 20, 1e-3, seed=9, dtype=dtype)
    omega = ref_cpu.normal_sketch(800, 30, 0, dtype=dtype)
    f = rsvd_incore(A, SketchConfig(20, 10, 2), omega=omega)
    fp64 = dtype == np.float64
    np.testing.assert_allclose(parts[0]["sigma"][:20], f.sigma[:20],
                               rtol=1e-10 if fp64 else 1e-5)
    np.testing.assert_allclose(U[:, :20], f.U[:, :20], atol=1e-8 if fp64 else 1e-3)
    np.testing.assert_allclose(parts[0]["Vt"][:20], f.Vt[:20], atol=1e-8 if fp64 else 1e-3)
    np.testing.assert_array_equal(parts[0]["sigma"], parts[1]["sigma"])


def test_library_nccl_communicator_world1():
    """The sharded driver over the library's own NCCL communicator
    (brsvd_ctx_attach_nccl / brsvd_allreduce / brsvd_allgather), one rank,
    against the single-GPU decomposition; a collective without a communicator
    fails as BRSVD_ERR_NCCL."""
    import ctypes
    import torch
    from oracle import ref_cpu
    from paper_1706_07191_b200 import SketchConfig, _lib, rsvd_incore
    from paper_1706_07191_b200.distributed import GpuOps, NcclComm, rsvd_sharded
    A = ref_cpu.lowrank_plus_noise(2000, 600, 20, 1e-3, seed=19, dtype=np.float64)
    omega = ref_cpu.normal_sketch(600, 30, 0, dtype=np.float64)
    fresh = ctypes.c_void_p()
    lib = _lib.load_library()
    assert lib.brsvd_ctx_create(0, None, ctypes.byref(fresh)) == _lib.OK
    buf = torch.zeros(4, dtype=torch.float64, device="cuda")
    assert lib.brsvd_allreduce(fresh, ctypes.c_void_p(buf.data_ptr()), 4, 1, 0) == _lib.ERR_NCCL
    lib.brsvd_ctx_destroy(fresh)
    ops = GpuOps(0)
    comm = NcclComm(ops)
    f, _ = rsvd_sharded(torch.as_tensor(A, device="cuda"), SketchConfig(20, 10, 2), 0, 2000,
                        comm=comm, ops=ops, omega=omega)
    ref = rsvd_incore(A, SketchConfig(20, 10, 2), omega=omega)
    np.testing.assert_allclose(f.sigma.cpu().numpy()[:20], ref.sigma[:20], rtol=1e-10)
    np.testing.assert_allclose(f.U.cpu().numpy()[:, :20], ref.U[:, :20], atol=1e-8)


@pytest.mark.parametrize("dtype", [np.float64, np.float32])
@pytest.mark.parametrize("q", [1, 2])
@pytest.mark.parametrize("frac", [0.99, 1.01])
def test_sharded_overflow_guard_exact_on_gpu(dtype, q, frac):
    """The sharded driver's exact _check_overflow (rsvd.py:84-91) through the
    C ABI (brsvd_normalize_t / brsvd_unnormalised_peak): fires iff the
    reference's unnormalised sample peaks above 0.01 * finfo.max."""
    import torch
    from oracle import ref_cpu
    from paper_1706_07191_b200 import SketchConfig
    from paper_1706_07191_b200.distributed import GpuOps, TorchComm, rsvd_sharded
    a = ref_cpu.lowrank_plus_noise(300, 200, 5, 1e-2, seed=8)
    omega = ref_cpu.normal_sketch(200, 10, 0, dtype=np.float64)
    peak1 = float(np.max(np.abs(ref_cpu.power_sample(a, omega, q))))
    lim = 0.01 * float(np.finfo(dtype).max)
    c = (frac * lim / peak1) ** (1.0 / (2 * q + 1))
    ac = (a * c).astype(dtype)
    om = omega.astype(dtype)
    with np.errstate(over="ignore", invalid="ignore"):
        _, ref_fires = ref_cpu.overflow_peak(ref_cpu.power_sample(ac, om, q))
    assert ref_fires == (frac > 1.0)
    A = torch.as_tensor(ac, device="cuda")
    if ref_fires:
        with pytest.raises(FloatingPointError):
            rsvd_sharded(A, SketchConfig(5, 5, q), 0, 300, comm=TorchComm(), ops=GpuOps(0),
                         omega=om)
    else:
        f, _ = rsvd_sharded(A, SketchConfig(5, 5, q), 0, 300, comm=TorchComm(), ops=GpuOps(0),
                            omega=om)
        assert np.isfinite(f.sigma.cpu().numpy()).all()
