"""The multi-GPU z-slab path's host logic on CPU: world_size 2 over gloo.

Each rank owns a z-slab (``dist.SlabDomain``), runs the oracle's line-Jacobi
sweep on its slab (standing in for the CUDA kernel, which needs a GPU), and
uses the product's exchange code (``start_exchange`` / ``finish_exchange``,
``gather_plane_sums``) for the halo planes and the history.  The assembled
result must equal the single-domain oracle bit for bit (Jacobi slab splits
are exact), history included."""

import math
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from oracle import restate as R

SHAPE = (24, 10, 12)
STEPS = 4
OMEGA = 0.8


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _fview(t):
    return t.numpy().transpose(2, 1, 0)  # F-ordered (px, py, pz) view


def _inputs():
    rng = np.random.default_rng(17)
    return rng.standard_normal(SHAPE), rng.standard_normal(SHAPE)


def _rank_main(rank, world, port, out_dir):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_1208_1975_b200.dist import SlabDomain, gather_plane_sums

        dom = SlabDomain(SHAPE, rank, world, device="cpu")
        u0, f = _inputs()
        p = dom.patch
        p.interior[...] = torch.from_numpy(np.ascontiguousarray(u0[:, :, dom.k0:dom.k1]))
        p.f[...] = torch.from_numpy(np.ascontiguousarray(f[:, :, dom.k0:dom.k1]))
        fl = _fview(p._f)

        def refresh():
            u = _fview(p._bufs[p._active])
            R.fill_physical_ghosts(u)
            reqs = dom.start_exchange(p._active)
            dom.finish_exchange(reqs)
            if dom.lo_rank is not None:
                u[1:-1, 1:-1, 0] = _fview(dom.stage_lo[None])[1:-1, 1:-1, 0]
            if dom.hi_rank is not None:
                u[1:-1, 1:-1, -1] = _fview(dom.stage_hi[None])[1:-1, 1:-1, 0]

        def plane_sums():
            u = _fview(p._bufs[p._active])
            r = R.residual(u, fl)
            return np.array([np.sum(np.square(r[:, :, k])) for k in range(dom.nz_local)])

        refresh()
        sums = []
        for _ in range(STEPS):
            u = _fview(p._bufs[p._active])
            v = _fview(p._bufs[1 - p._active])
            sums.append(plane_sums())
            r = R.residual(u, fl)
            v[1:-1, 1:-1, 1:-1] = u[1:-1, 1:-1, 1:-1] + OMEGA * R.line_solve(r)
            p.swap_buffers()
            refresh()
        sums.append(plane_sums())
        full = gather_plane_sums(torch.from_numpy(np.stack(sums)))
        hist = [math.sqrt(float(np.sum(row))) for row in full.numpy()]
        np.save(os.path.join(out_dir, f"slab{rank}.npy"), p.interior.numpy())
        np.save(os.path.join(out_dir, f"hist{rank}.npy"), np.array(hist))
        dist.barrier()
    finally:
        dist.destroy_process_group()


def test_two_rank_slab_jacobi_equals_single_domain(tmp_path):
    world = 2
    mp.spawn(_rank_main, args=(world, _free_port(), str(tmp_path)), nprocs=world, join=True)
    u0, f = _inputs()
    o = R.OPatch(SHAPE)
    o.u[1:-1, 1:-1, 1:-1] = u0
    o.f[:] = f
    lv = R.OLevel([o])
    lv.refresh_ghosts()
    want_hist = []
    for _ in range(STEPS):
        r = R.residual(o.u, o.f)
        want_hist.append(math.sqrt(sum(np.sum(np.square(r[:, :, k])) for k in range(SHAPE[2]))))
        R.jacobi_step(lv, (SHAPE[0], 1, 1), OMEGA)
    r = R.residual(o.u, o.f)
    want_hist.append(math.sqrt(sum(np.sum(np.square(r[:, :, k])) for k in range(SHAPE[2]))))
    got = np.concatenate([np.load(tmp_path / f"slab{r}.npy") for r in range(world)], axis=2)
    np.testing.assert_array_equal(got, o.interior)
    for r in range(world):
        h = np.load(tmp_path / f"hist{r}.npy")
        np.testing.assert_allclose(h, want_hist, rtol=1e-14, atol=0)
    np.testing.assert_array_equal(np.load(tmp_path / "hist0.npy"), np.load(tmp_path / "hist1.npy"))


@pytest.mark.parametrize("nz,world", [(12, 2), (13, 4), (1024, 8), (9, 3)])
def test_slab_ranges_tile_the_grid(nz, world):
    from paper_1208_1975_b200.dist import slab_range

    spans = [slab_range(nz, world, r) for r in range(world)]
    assert spans[0][0] == 0 and spans[-1][1] == nz
    assert all(a[1] == b[0] for a, b in zip(spans, spans[1:]))
    sizes = [b - a for a, b in spans]
    assert max(sizes) - min(sizes) <= 1


def _level_main(rank, world, port, out_dir):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_1208_1975_b200.dist import PatchLevelDomain

        specs = [((4, 3, 2), (a * 4, b * 3, c * 2)) for c in range(2) for b in range(2) for a in range(3)]
        dom = PatchLevelDomain(specs, rank, world, device="cpu")
        for g, p in zip(dom.mine, dom.patches):
            p.u[...] = -1.0
            p.interior[...] = torch.arange(24, dtype=torch.float64).reshape(4, 3, 2) + 100.0 * g
        dom.exchange()
        for g, p in zip(dom.mine, dom.patches):
            np.save(os.path.join(out_dir, f"u{g}.npy"), p.u.numpy())
        np.save(os.path.join(out_dir, f"owner{rank}.npy"), np.array(dom.mine))
        dist.barrier()
    finally:
        dist.destroy_process_group()


def test_patch_partition_exchange_fills_cross_rank_ghosts(tmp_path):
    """PatchLevelDomain: greedy patch-to-rank map, and exchange() writes every
    cross-rank ghost layer with the neighbour's interior layer (what the
    device refresh does for same-rank pairs)."""
    from paper_1208_1975_b200.dist import PatchLevelDomain, _PatchSpec
    from paper_1208_1975_b200.grid import _abutments

    world = 3
    mp.spawn(_level_main, args=(world, _free_port(), str(tmp_path)), nprocs=world, join=True)
    owned = sorted(int(g) for r in range(world) for g in np.load(tmp_path / f"owner{r}.npy"))
    assert owned == list(range(12))
    specs = [((4, 3, 2), (a * 4, b * 3, c * 2)) for c in range(2) for b in range(2) for a in range(3)]
    owner = {}
    for r in range(world):
        for g in np.load(tmp_path / f"owner{r}.npy"):
            owner[int(g)] = r
    adj = _abutments([_PatchSpec(d, o) for d, o in specs])
    checked = 0
    for c in adj:
        if owner[c.src] == owner[c.dst]:
            continue
        src = np.load(tmp_path / f"u{c.src}.npy")
        dst = np.load(tmp_path / f"u{c.dst}.npy")
        s = tuple(slice(1 + lo, 1 + lo + e) for lo, e in zip(c.src_lo, c.extent))
        d = tuple(slice(1 + lo, 1 + lo + e) for lo, e in zip(c.dst_lo, c.extent))
        np.testing.assert_array_equal(dst[d], src[s])
        checked += 1
    assert checked > 0


def test_slab_domain_halo_modes():
    from paper_1208_1975_b200.dist import SlabDomain

    d = SlabDomain((8, 4, 6), rank=1, world=2, device="cpu", halo="p2p")
    assert d.halo == "p2p" and d._peer is None and (d.k0, d.k1) == (3, 6)
    with pytest.raises(ValueError):
        SlabDomain((8, 4, 6), rank=0, world=2, device="cpu", halo="shm")


def _ragged_main(rank, world, port, out_dir):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_1208_1975_b200.dist import gather_plane_sums, slab_range

        k0, k1 = slab_range(17, world, rank)
        local = torch.arange(k0, k1, dtype=torch.float64)[None, :].repeat(2, 1) + 100.0 * torch.arange(2)[:, None]
        full = gather_plane_sums(local)
        np.save(os.path.join(out_dir, f"g{rank}.npy"), full.numpy())
    finally:
        dist.destroy_process_group()


def test_gather_plane_sums_ragged_slabs(tmp_path):
    """17 planes over 3 ranks (6, 6, 5): the gathered per-plane vector is the
    global one in plane order, no padding left in it."""
    world = 3
    mp.spawn(_ragged_main, args=(world, _free_port(), str(tmp_path)), nprocs=world, join=True)
    want = np.arange(17, dtype=np.float64)[None, :] + 100.0 * np.arange(2)[:, None]
    for r in range(world):
        np.testing.assert_array_equal(np.load(tmp_path / f"g{r}.npy"), want)


def test_patch_level_domain_halo_modes():
    from paper_1208_1975_b200.dist import PatchLevelDomain

    specs = [((8, 4, 4), (0, 0, 0)), ((8, 4, 4), (8, 0, 0))]
    d = PatchLevelDomain(specs, 0, 2, device="cpu", halo="p2p")
    assert d.halo == "p2p" and d._peer is None
    with pytest.raises(ValueError):
        PatchLevelDomain(specs, 0, 2, device="cpu", halo="ucx")
