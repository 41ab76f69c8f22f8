"""Two ranks on two different GPUs (one process per device, NCCL): the
z-slab line-Jacobi path with the halo over NCCL and with the fused
peer-memory halo (CUDA IPC across devices, gated on cudaDeviceCanAccessPeer)
must equal the single-process run bit for bit, history included.
Skipped when fewer than two GPUs are visible (the round-end boxes have one;
the 8-GPU node runs it)."""

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

pytestmark = [pytest.mark.gpu,
              pytest.mark.skipif(torch.cuda.device_count() < 2, reason="needs two visible GPUs")]
SHAPE = (256, 40, 24)
STEPS = 4


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _inputs():
    rng = np.random.default_rng(31)
    return rng.standard_normal(SHAPE), rng.standard_normal(SHAPE)


def _rank_main(rank, world, port, out_dir, halo):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    torch.cuda.set_device(rank)
    dist.init_process_group("nccl", rank=rank, world_size=world, device_id=torch.device("cuda", rank))
    try:
        import paper_1208_1975_b200 as ps
        from paper_1208_1975_b200.dist import SlabDomain, dist_smooth

        dom = SlabDomain(SHAPE, rank, world, device=f"cuda:{rank}", halo=halo)
        u0, f = _inputs()
        p = dom.patch
        p.interior[...] = torch.from_numpy(np.ascontiguousarray(u0[:, :, dom.k0:dom.k1])).to(p.device)
        p.f[...] = torch.from_numpy(np.ascontiguousarray(f[:, :, dom.k0:dom.k1])).to(p.device)
        cfg = ps.SmootherConfig(scheme="block_jacobi", block_dims=(SHAPE[0], 1, 1), steps=STEPS,
                                strategy=ps.ExecutionStrategy.device(devices=world))
        hist = dist_smooth(dom, cfg, ps.InverseCache())
        np.save(os.path.join(out_dir, f"slab{rank}.npy"), p.interior.cpu().numpy())
        np.save(os.path.join(out_dir, f"hist{rank}.npy"), np.array(hist))
        dist.barrier()
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("halo", ["nccl", "p2p"])
def test_two_devices_match_single_process(tmp_path, halo):
    import paper_1208_1975_b200 as ps

    world = 2
    mp.spawn(_rank_main, args=(world, _free_port(), str(tmp_path), halo), nprocs=world, join=True)
    u0, f = _inputs()
    p = ps.Patch(ps.PatchDims(*SHAPE), device="cuda:0")
    p.interior[...] = torch.from_numpy(u0).cuda()
    p.f[...] = torch.from_numpy(f).cuda()
    cfg = ps.SmootherConfig(scheme="block_jacobi", block_dims=(SHAPE[0], 1, 1), steps=STEPS)
    _, want = ps.smooth(ps.Level([p]), cfg, ps.InverseCache())
    got = np.concatenate([np.load(tmp_path / f"slab{r}.npy") for r in range(world)], axis=2)
    np.testing.assert_array_equal(got, p.interior.cpu().numpy())
    for r in range(world):
        np.testing.assert_array_equal(np.load(tmp_path / f"hist{r}.npy"), np.array(want))
