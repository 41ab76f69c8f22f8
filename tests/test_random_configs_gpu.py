"""Randomised configurations against the CPU restatement: patch shapes
(including 1-wide axes and odd sizes), line / plane / box blocks, Jacobi and
GS, omega, non-default stencils and 1-3 patch levels.  Every case within
1e-12 relative max-norm (iterates with ghosts, history)."""

import numpy as np
import pytest
import torch

import golden_io as G
import paper_1208_1975_b200 as ps
from oracle import restate as R

pytestmark = pytest.mark.gpu

STENCILS = [(6.0, (-1.0,) * 6), (7.0, (-1.3, -0.7, -1.1, -0.9, -1.0, -1.2)),
            (6.5, (-1.2, -1.2, -0.8, -1.1, -0.9, -1.0)), (4.2, (-1.0, -1.0, -0.5, -0.5, 0.0, 0.0))]


def _case(seed):
    rng = np.random.default_rng(1000 + seed)
    kind = ["line", "plane", "box"][seed % 3]
    scheme = ["block_jacobi", "chaotic_block_gs"][(seed // 3) % 2]
    center, faces = STENCILS[seed % len(STENCILS)]
    if kind == "plane" and faces[0] != faces[1]:
        center, faces = STENCILS[2]
    if kind == "box" and any(a * b < 0 for a, b in zip(faces[0::2], faces[1::2])):
        center, faces = STENCILS[0]
    nx = int(rng.choice([1, 3, 8, 17, 32, 64, 100, 128]))
    ny = int(rng.integers(1, 12))
    nz = int(rng.integers(1, 10))
    npatch = int(rng.integers(1, 4))
    if kind == "line":
        block = (nx, 1, 1)
    elif kind == "plane":
        block = (nx, ny, 1)
    else:
        block = tuple(int(b) for b in rng.integers(1, 9, size=3))
    omega = 0.7 if rng.random() < 0.4 else None
    return kind, scheme, (center, faces), (nx, ny, nz), npatch, block, omega


@pytest.mark.parametrize("seed", range(36))
def test_random_configuration(seed):
    kind, scheme, (center, faces), shape, npatch, block, omega = _case(seed)
    rng = np.random.default_rng(seed)
    ops, gps = [], []
    for i in range(npatch):
        u0, f = rng.standard_normal(shape), rng.standard_normal(shape)
        o = R.OPatch(shape, (i * shape[0], 0, 0))
        o.u[1:-1, 1:-1, 1:-1] = u0
        o.f[:] = f
        g = ps.Patch(ps.PatchDims(*shape), (i * shape[0], 0, 0))
        g.interior[...] = torch.from_numpy(u0).cuda()
        g.f[...] = torch.from_numpy(f).cuda()
        ops.append(o)
        gps.append(g)
    o, g = R.OLevel(ops), ps.Level(gps)
    want = R.smooth(o, scheme, block, omega=omega, steps=2, center=center, faces=faces, exact_norm=False)
    cfg = ps.SmootherConfig(scheme=scheme, block_dims=block, omega=omega, steps=2, stencil=ps.Stencil7(center, faces))
    _, hist = ps.smooth(g, cfg, ps.InverseCache())
    for po, pg in zip(o.patches, g.patches):
        assert G.rel_maxnorm(pg.u.cpu().numpy(), po.u) < 1e-12, (kind, scheme, shape, block)
    assert G.hist_rel(hist, want) < 1e-12
