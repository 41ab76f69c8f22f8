"""The multi-process z-slab path with the real CUDA kernels: two ranks on
one GPU (gloo, halo planes staged through host memory -- the driver's boxes
have one GPU; NCCL itself needs one GPU per rank).  Line Jacobi on slabs must
equal the single-patch run bit for bit, history included; GS on
slabs must equal GS on the same split level run in one process."""

import math
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

pytestmark = pytest.mark.gpu
SHAPE = (128, 24, 14)
STEPS = 3


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _inputs():
    rng = np.random.default_rng(23)
    return rng.standard_normal(SHAPE), rng.standard_normal(SHAPE)


def _rank_main(rank, world, port, out_dir, scheme):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import paper_1208_1975_b200 as ps
        from paper_1208_1975_b200.dist import SlabDomain, dist_smooth

        torch.cuda.set_device(0)
        dom = SlabDomain(SHAPE, rank, world, device="cuda:0")
        u0, f = _inputs()
        p = dom.patch
        p.interior[...] = torch.from_numpy(np.ascontiguousarray(u0[:, :, dom.k0:dom.k1])).cuda()
        p.f[...] = torch.from_numpy(np.ascontiguousarray(f[:, :, dom.k0:dom.k1])).cuda()
        cfg = ps.SmootherConfig(scheme=scheme, block_dims=(SHAPE[0], 1, 1), steps=STEPS,
                                strategy=ps.ExecutionStrategy.device(devices=world))
        hist = dist_smooth(dom, cfg, ps.InverseCache())
        np.save(os.path.join(out_dir, f"slab{rank}.npy"), p.interior.cpu().numpy())
        np.save(os.path.join(out_dir, f"hist{rank}.npy"), np.array(hist))
        dist.barrier()
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("scheme", ["block_jacobi", "chaotic_block_gs"])
def test_two_rank_slabs_match_single_process(tmp_path, scheme):
    import paper_1208_1975_b200 as ps
    from paper_1208_1975_b200.dist import slab_range

    world = 2
    mp.spawn(_rank_main, args=(world, _free_port(), str(tmp_path), scheme), nprocs=world, join=True)
    u0, f = _inputs()
    if scheme == "block_jacobi":  # one patch: the split is exact
        patches = [ps.Patch(ps.PatchDims(*SHAPE))]
        spans = [(0, SHAPE[2])]
    else:  # GS on slabs == GS on the same split level
        spans = [slab_range(SHAPE[2], world, r) for r in range(world)]
        patches = [ps.Patch(ps.PatchDims(SHAPE[0], SHAPE[1], b - a), (0, 0, a)) for a, b in spans]
    for p, (a, b) in zip(patches, spans):
        p.interior[...] = torch.from_numpy(np.ascontiguousarray(u0[:, :, a:b])).cuda()
        p.f[...] = torch.from_numpy(np.ascontiguousarray(f[:, :, a:b])).cuda()
    lv = ps.Level(patches)
    cfg = ps.SmootherConfig(scheme=scheme, block_dims=(SHAPE[0], 1, 1), steps=STEPS,
                            strategy=ps.ExecutionStrategy.device())
    _, want_hist = ps.smooth(lv, cfg, ps.InverseCache())
    want = np.concatenate([p.interior.cpu().numpy() for p in patches], axis=2)
    got = np.concatenate([np.load(tmp_path / f"slab{r}.npy") for r in range(world)], axis=2)
    if scheme == "block_jacobi":
        np.testing.assert_array_equal(got, want)
        for r in range(world):
            np.testing.assert_array_equal(np.load(tmp_path / f"hist{r}.npy"), np.array(want_hist))
    else:
        assert np.max(np.abs(got - want)) / np.max(np.abs(want)) < 1e-12
        for r in range(world):
            h = np.load(tmp_path / f"hist{r}.npy")
            assert max(abs(a - b) / b for a, b in zip(h, want_hist)) < 1e-12


LATTICE = (2, 2, 2)
PSIZE = (64, 8, 6)


def _lattice_specs():
    return [(PSIZE, (a * PSIZE[0], b * PSIZE[1], c * PSIZE[2]))
            for c in range(LATTICE[2]) for b in range(LATTICE[1]) for a in range(LATTICE[0])]


def _lattice_inputs():
    rng = np.random.default_rng(31)
    n = LATTICE[0] * LATTICE[1] * LATTICE[2]
    return [rng.standard_normal(PSIZE) for _ in range(n)], [rng.standard_normal(PSIZE) for _ in range(n)]


def _level_rank_main(rank, world, port, out_dir, scheme, block):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import paper_1208_1975_b200 as ps
        from paper_1208_1975_b200.dist import PatchLevelDomain, dist_smooth_level

        torch.cuda.set_device(0)
        dom = PatchLevelDomain(_lattice_specs(), rank, world, device="cuda:0")
        u0, f = _lattice_inputs()
        for g, p in zip(dom.mine, dom.patches):
            p.interior[...] = torch.from_numpy(u0[g]).cuda()
            p.f[...] = torch.from_numpy(f[g]).cuda()
        cfg = ps.SmootherConfig(scheme=scheme, block_dims=block, steps=STEPS)
        hist = dist_smooth_level(dom, cfg, ps.InverseCache())
        for g, p in zip(dom.mine, dom.patches):
            np.save(os.path.join(out_dir, f"patch{g}.npy"), p.u.cpu().numpy())
        np.save(os.path.join(out_dir, f"lhist{rank}.npy"), np.array(hist))
        dist.barrier()
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("scheme,block", [("block_jacobi", (64, 1, 1)), ("chaotic_block_gs", (64, 1, 1)),
                                          ("block_jacobi", (4, 4, 2)), ("chaotic_block_gs", (64, 8, 1))])
def test_two_rank_patch_partition_matches_single_process(tmp_path, scheme, block):
    """C4-style lattice split by patch over 2 ranks (cross-rank interface
    copies packed/sent/unpacked): bitwise equal to the single-process level,
    iterates (ghosts included) and history."""
    import paper_1208_1975_b200 as ps

    world = 2
    mp.spawn(_level_rank_main, args=(world, _free_port(), str(tmp_path), scheme, block), nprocs=world, join=True)
    u0, f = _lattice_inputs()
    patches = [ps.Patch(ps.PatchDims(*d), o) for d, o in _lattice_specs()]
    for p, a, b in zip(patches, u0, f):
        p.interior[...] = torch.from_numpy(a).cuda()
        p.f[...] = torch.from_numpy(b).cuda()
    lv = ps.Level(patches)
    cfg = ps.SmootherConfig(scheme=scheme, block_dims=block, steps=STEPS)
    _, want_hist = ps.smooth(lv, cfg, ps.InverseCache())
    for g, p in enumerate(patches):
        np.testing.assert_array_equal(np.load(tmp_path / f"patch{g}.npy"), p.u.cpu().numpy())
    for r in range(world):
        np.testing.assert_array_equal(np.load(tmp_path / f"lhist{r}.npy"), np.array(want_hist))
