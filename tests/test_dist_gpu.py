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

import golden_io as G
from oracle import restate as R

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


def _level_rank_main(rank, world, port, out_dir, scheme, block, halo="nccl"):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import paper_1208_1975_b200 as ps
        from paper_1208_1975_b200.dist import PatchLevelDomain, dist_smooth_level

        torch.cuda.set_device(0)
        dom = PatchLevelDomain(_lattice_specs(), rank, world, device="cuda:0", halo=halo)
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


@pytest.mark.parametrize("scheme,block,halo", [("block_jacobi", (64, 1, 1), "nccl"),
                                               ("chaotic_block_gs", (64, 1, 1), "nccl"),
                                               ("block_jacobi", (4, 4, 2), "nccl"),
                                               ("chaotic_block_gs", (64, 8, 1), "nccl"),
                                               ("block_jacobi", (64, 1, 1), "p2p"),
                                               ("chaotic_block_gs", (64, 8, 1), "p2p")])
def test_two_rank_patch_partition_matches_single_process(tmp_path, scheme, block, halo):
    """C4-style lattice split by patch over 2 ranks (cross-rank interface
    copies packed/sent/unpacked): bitwise equal to the single-process level,
    iterates (ghosts included) and history."""
    import paper_1208_1975_b200 as ps

    world = 2
    mp.spawn(_level_rank_main, args=(world, _free_port(), str(tmp_path), scheme, block, halo), nprocs=world,
             join=True)
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


P2P_SHAPE = (128, 20, 17)  # three ragged slabs (6, 6, 5 planes); ny not a multiple of the tile rows


def _p2p_inputs():
    rng = np.random.default_rng(41)
    return rng.standard_normal(P2P_SHAPE), rng.standard_normal(P2P_SHAPE)


def _p2p_rank_main(rank, world, port, out_dir, calls):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import paper_1208_1975_b200 as ps
        from paper_1208_1975_b200.dist import SlabDomain, dist_smooth

        torch.cuda.set_device(0)
        dom = SlabDomain(P2P_SHAPE, rank, world, device="cuda:0", halo="p2p")
        u0, f = _p2p_inputs()
        p = dom.patch
        p.interior[...] = torch.from_numpy(np.ascontiguousarray(u0[:, :, dom.k0:dom.k1])).cuda()
        p.f[...] = torch.from_numpy(np.ascontiguousarray(f[:, :, dom.k0:dom.k1])).cuda()
        cfg = ps.SmootherConfig(scheme="block_jacobi", block_dims=(P2P_SHAPE[0], 1, 1), steps=STEPS, omega=0.8,
                                strategy=ps.ExecutionStrategy.device(devices=world))
        cache = ps.InverseCache()
        hists = [dist_smooth(dom, cfg, cache) for _ in range(calls)]
        assert dom._peer is not None and dom._peer.epoch == calls * STEPS
        np.save(os.path.join(out_dir, f"slab{rank}.npy"), p.u.cpu().numpy())
        np.save(os.path.join(out_dir, f"hist{rank}.npy"), np.array(hists))
        dist.barrier()
    finally:
        dist.destroy_process_group()


def _p2p_single_main(rank, out_dir, calls):
    os.environ["PSM_ZMARCH_MIN_CELLS"] = "0"
    import paper_1208_1975_b200 as ps

    torch.cuda.set_device(0)
    u0, f = _p2p_inputs()
    patch = ps.Patch(ps.PatchDims(*P2P_SHAPE))
    patch.interior[...] = torch.from_numpy(u0).cuda()
    patch.f[...] = torch.from_numpy(f).cuda()
    cfg = ps.SmootherConfig(scheme="block_jacobi", block_dims=(P2P_SHAPE[0], 1, 1), steps=STEPS, omega=0.8,
                            strategy=ps.ExecutionStrategy.device())
    cache = ps.InverseCache()
    hists = [ps.smooth(ps.Level([patch]), cfg, cache)[1] for _ in range(calls)]
    np.save(os.path.join(out_dir, "single.npy"), patch.u.cpu().numpy())
    np.save(os.path.join(out_dir, "single_hist.npy"), np.array(hists))


def _oracle_jacobi(u0, f, steps):
    o = R.OPatch(P2P_SHAPE)
    o.u[1:-1, 1:-1, 1:-1] = u0
    o.f[:] = f
    R.smooth(R.OLevel([o]), "block_jacobi", (P2P_SHAPE[0], 1, 1), omega=0.8, steps=steps)
    return o.u[1:-1, 1:-1, 1:-1]


def test_fused_peer_halo_matches_single_process(tmp_path):
    """The fused halo (the sweep stores its boundary planes into the
    neighbours' ghost planes over CUDA IPC, step flags instead of a
    collective): three ranks, ragged slabs, two consecutive smooth() calls --
    every iterate cell, ghosts included, and both histories bitwise equal to
    the single-patch run."""
    import paper_1208_1975_b200 as ps
    from paper_1208_1975_b200.dist import slab_range

    world, calls = 3, 2
    mp.spawn(_p2p_rank_main, args=(world, _free_port(), str(tmp_path), calls), nprocs=world, join=True)
    # the single-patch run in a child process with the z-marching kernel forced
    # too (the slabs run it whatever their size), so the arithmetic is the same
    mp.spawn(_p2p_single_main, args=(str(tmp_path), calls), nprocs=1, join=True)
    want = np.load(tmp_path / "single.npy")
    want_hists = np.load(tmp_path / "single_hist.npy")
    u0, f = _p2p_inputs()
    assert G.rel_maxnorm(want[1:-1, 1:-1, 1:-1], _oracle_jacobi(u0, f, calls * STEPS)) < 1e-12
    for r in range(world):
        k0, k1 = slab_range(P2P_SHAPE[2], world, r)
        got = np.load(tmp_path / f"slab{r}.npy")  # padded (x, y, z) incl. ghosts
        np.testing.assert_array_equal(got[1:-1, 1:-1, :], want[1:-1, 1:-1, k0:k1 + 2])
        np.testing.assert_array_equal(np.load(tmp_path / f"hist{r}.npy"), np.array(want_hists))


# a mixed-size patch set with partial-face abutment across ranks
MIXED_SPECS = [((16, 12, 10), (0, 0, 0)), ((20, 12, 10), (16, 0, 0)), ((12, 8, 6), (36, 2, 1)),
               ((24, 16, 12), (0, 12, 0)), ((16, 16, 16), (24, 12, 0)), ((8, 20, 14), (40, 10, 2)),
               ((32, 10, 8), (0, 0, 10))]


def _mixed_inputs():
    rng = np.random.default_rng(53)
    return [rng.standard_normal(d) for d, _ in MIXED_SPECS], [rng.standard_normal(d) for d, _ in MIXED_SPECS]


def _mixed_rank_main(rank, world, port, out_dir, scheme, block, halo="nccl"):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import paper_1208_1975_b200 as ps
        from paper_1208_1975_b200.dist import PatchLevelDomain, dist_smooth_level

        torch.cuda.set_device(0)
        dom = PatchLevelDomain(MIXED_SPECS, rank, world, device="cuda:0", halo=halo)
        u0, f = _mixed_inputs()
        for g, p in zip(dom.mine, dom.patches):
            p.interior[...] = torch.from_numpy(u0[g]).cuda()
            p.f[...] = torch.from_numpy(f[g]).cuda()
        cfg = ps.SmootherConfig(scheme=scheme, block_dims=block, steps=STEPS)
        cache = ps.InverseCache()
        hist = dist_smooth_level(dom, cfg, cache)
        if halo == "p2p":  # the peer path really ran, and a second call continues the flag epochs
            assert dom._peer is not None and dom._peer.epoch == STEPS
            hist2 = dist_smooth_level(dom, cfg, cache)
            np.save(os.path.join(out_dir, f"mhist2_{rank}.npy"), np.array(hist2))
        for g, p in zip(dom.mine, dom.patches):
            np.save(os.path.join(out_dir, f"patch{g}.npy"), p.u.cpu().numpy())
        np.save(os.path.join(out_dir, f"mhist{rank}.npy"), np.array(hist))
        dist.barrier()
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("scheme,block,halo", [("block_jacobi", (32, 1, 1), "nccl"),
                                               ("chaotic_block_gs", (32, 1, 1), "nccl"),
                                               ("block_jacobi", (4, 4, 4), "nccl"),
                                               ("block_jacobi", (32, 1, 1), "p2p"),
                                               ("chaotic_block_gs", (32, 1, 1), "p2p"),
                                               ("block_jacobi", (4, 4, 4), "p2p"),
                                               ("block_jacobi", (32, 32, 1), "p2p")])
def test_mixed_patch_set_across_three_ranks(tmp_path, scheme, block, halo):
    """Seven patches of different sizes (partial-face abutment on every axis,
    some faces physical, some shared with two patches) split greedily over 3
    ranks: bitwise equal to the single-process level, ghosts and history.
    halo='p2p': the cross-rank faces are pulled from the neighbours' memory
    (CUDA IPC) by one copy launch per step, step flags instead of NCCL; two
    consecutive calls."""
    import paper_1208_1975_b200 as ps

    world = 3
    mp.spawn(_mixed_rank_main, args=(world, _free_port(), str(tmp_path), scheme, block, halo), nprocs=world,
             join=True)
    u0, f = _mixed_inputs()
    patches = [ps.Patch(ps.PatchDims(*d), o) for d, o in MIXED_SPECS]
    for p, a, b in zip(patches, u0, f):
        p.interior[...] = torch.from_numpy(a).cuda()
        p.f[...] = torch.from_numpy(b).cuda()
    lv = ps.Level(patches)
    assert len(lv.adjacency) >= len(MIXED_SPECS)  # the layout really has shared (partial) faces
    cfg = ps.SmootherConfig(scheme=scheme, block_dims=block, steps=STEPS)
    cache = ps.InverseCache()
    _, want_hist = ps.smooth(lv, cfg, cache)
    if halo == "p2p":
        _, want_hist2 = ps.smooth(lv, cfg, cache)
    for g, p in enumerate(patches):
        np.testing.assert_array_equal(np.load(tmp_path / f"patch{g}.npy"), p.u.cpu().numpy())
    for r in range(world):
        np.testing.assert_array_equal(np.load(tmp_path / f"mhist{r}.npy"), np.array(want_hist))
        if halo == "p2p":
            np.testing.assert_array_equal(np.load(tmp_path / f"mhist2_{r}.npy"), np.array(want_hist2))
