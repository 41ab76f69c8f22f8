"""The hand-written DMMA DST-I transforms of the plane path
(psm_plane_dst.cu: parity-split tiles with fused residual / relaxation) and
the one-launch plane-GS stage chain, against the CPU restatement: the exact
plane inverse applied to random blocks (BlockFactors.apply), plane Jacobi in
'dst' mode, and plane GS on single patches, lattices and mixed odd/even
patch sizes (unaligned workspace offsets).  Tolerance 1e-12 relative."""

import numpy as np
import pytest
import torch

import golden_io as G
import paper_1208_1975_b200 as ps
from oracle import restate as R

pytestmark = pytest.mark.gpu
TOL = 1e-12


def _pair(shapes_origins, seed):
    rng = np.random.default_rng(seed)
    ops, gps = [], []
    for shape, origin in shapes_origins:
        u0, f = rng.standard_normal(shape), rng.standard_normal(shape)
        o = R.OPatch(shape, origin)
        o.u[1:-1, 1:-1, 1:-1] = u0
        o.f[:] = f
        g = ps.Patch(ps.PatchDims(*shape), origin)
        g.interior[...] = torch.from_numpy(u0).cuda()
        g.f[...] = torch.from_numpy(f).cuda()
        ops.append(o)
        gps.append(g)
    return R.OLevel(ops), ps.Level(gps)


@pytest.mark.parametrize("nx,ny", [(1, 3), (2, 2), (3, 5), (5, 4), (8, 8), (31, 7), (64, 9), (100, 5), (128, 128),
                                   (129, 4), (200, 3), (256, 6), (300, 2), (511, 2), (512, 3)])
def test_plane_inverse_apply(nx, ny):
    rng = np.random.default_rng(nx * 1000 + ny)
    count = 3
    r = rng.standard_normal((count, ny, nx))  # blocks cells x fastest
    fac = ps.BlockFactors(ps.Stencil7(), (nx, ny, 1), "cuda")
    got = fac.apply(torch.from_numpy(r.reshape(count, nx * ny)).cuda()).cpu().numpy().reshape(count, ny, nx)
    for c in range(count):
        want = R.plane_solve(r[c].T[:, :, None])[:, :, 0].T  # restatement indexes (x, y, z)
        assert G.rel_maxnorm(got[c], want) < TOL


@pytest.mark.parametrize("shape", [(64, 48, 5), (100, 37, 3), (128, 128, 3), (33, 20, 4), (512, 40, 2)])
def test_dst_mode_plane_jacobi(shape):
    prev = ps.plane_solver("dst")
    try:
        o, g = _pair([(shape, (0, 0, 0))], seed=sum(shape))
        want = R.smooth(o, "block_jacobi", (shape[0], shape[1], 1), steps=2, exact_norm=False)
        cfg = ps.SmootherConfig(scheme="block_jacobi", block_dims=(shape[0], shape[1], 1), steps=2)
        _, hist = ps.smooth(g, cfg, ps.InverseCache())
    finally:
        ps.plane_solver(prev)
    assert G.rel_maxnorm(g.patches[0].u.cpu().numpy(), o.patches[0].u) < TOL
    assert G.hist_rel(hist, want) < TOL


@pytest.mark.parametrize("shape", [(128, 128, 9), (64, 64, 20), (77, 30, 6), (16, 1, 5), (5, 7, 3), (256, 12, 4)])
def test_plane_gs_single_patch(shape):
    o, g = _pair([(shape, (0, 0, 0))], seed=7 + sum(shape))
    block = (shape[0], shape[1], 1)
    want = R.smooth(o, "chaotic_block_gs", block, steps=2, exact_norm=False)
    _, hist = ps.smooth(g, ps.SmootherConfig(scheme="chaotic_block_gs", block_dims=block, steps=2),
                        ps.InverseCache())
    assert G.rel_maxnorm(g.patches[0].u.cpu().numpy(), o.patches[0].u) < TOL
    assert G.hist_rel(hist, want) < TOL


def test_plane_gs_mixed_odd_even_patches():
    """9^3 before 16^3: the 16^3 patch's workspace offset (cell0 = 729) is odd,
    so its planes are only 8-byte aligned (advisor finding, round 1)."""
    so = [((9, 9, 9), (0, 0, 0)), ((16, 16, 16), (9, 0, 0)), ((16, 16, 16), (0, 16, 0)), ((9, 9, 9), (25, 0, 0))]
    o, g = _pair(so, seed=3)
    want = R.smooth(o, "chaotic_block_gs", (16, 16, 1), steps=2, exact_norm=False)
    cfg = ps.SmootherConfig(scheme="chaotic_block_gs", block_dims=(16, 16, 1), steps=2)
    _, hist = ps.smooth(g, cfg, ps.InverseCache())
    for po, pg in zip(o.patches, g.patches):
        assert G.rel_maxnorm(pg.u.cpu().numpy(), po.u) < TOL
    assert G.hist_rel(hist, want) < TOL


def test_plane_gs_lattice_different_nz():
    so = [((32, 24, 7), (0, 0, 0)), ((32, 24, 3), (32, 0, 0)), ((32, 24, 11), (0, 24, 0))]
    o, g = _pair(so, seed=5)
    want = R.smooth(o, "chaotic_block_gs", (32, 24, 1), omega=0.9, steps=3, exact_norm=False)
    cfg = ps.SmootherConfig(scheme="chaotic_block_gs", block_dims=(32, 24, 1), omega=0.9, steps=3)
    _, hist = ps.smooth(g, cfg, ps.InverseCache())
    for po, pg in zip(o.patches, g.patches):
        assert G.rel_maxnorm(pg.u.cpu().numpy(), po.u) < TOL
    assert G.hist_rel(hist, want) < TOL
