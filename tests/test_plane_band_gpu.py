"""Parity of the banded factorised plane solve (psm_plane_band.cu) with the
CPU restatement (exact DST-I plane inverse) and with the device DST form:
iterates and histories within 1e-12 relative max-norm.  Shapes cover nx not
a multiple of the 64-thread CTA, ny beyond the converged Schur complement,
ny shorter than convergence, non-symmetric y faces, omega != default and
multi-patch lattices."""

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


def _run(o, g, scheme, steps, omega=None, center=6.0, faces=(-1.0,) * 6):
    d = g.patches[0].dims
    want = R.smooth(o, scheme, (d.nx, d.ny, 1), omega=omega, steps=steps, center=center, faces=faces,
                    exact_norm=False)
    cfg = ps.SmootherConfig(scheme=scheme, block_dims=(d.nx, d.ny, 1), omega=omega, steps=steps,
                            stencil=ps.Stencil7(center, faces))
    _, hist = ps.smooth(g, cfg, ps.InverseCache())
    return want, hist


@pytest.mark.parametrize("shape", [(64, 48, 5), (128, 128, 3), (100, 37, 3), (512, 40, 2), (96, 300, 2),
                                   (48, 5, 4), (17, 64, 3), (1000, 8, 1)])
def test_band_plane_jacobi_matches_restatement(shape):
    assert ps.plane_solver() == "auto"
    o, g = _pair([(shape, (0, 0, 0))], seed=sum(shape))
    want, hist = _run(o, g, "block_jacobi", steps=2)
    assert G.rel_maxnorm(g.patches[0].u.cpu().numpy(), o.patches[0].u) < TOL
    assert G.hist_rel(hist, want) < TOL


def test_band_plane_jacobi_nonsymmetric_y_faces_and_omega():
    center, faces = 6.4, (-1.1, -1.1, -0.7, -1.3, -1.0, -0.9)
    o, g = _pair([((96, 80, 3), (0, 0, 0))], seed=4)
    want, hist = _run(o, g, "block_jacobi", steps=3, omega=0.6, center=center, faces=faces)
    assert G.rel_maxnorm(g.patches[0].u.cpu().numpy(), o.patches[0].u) < TOL
    assert G.hist_rel(hist, want) < TOL


def test_band_plane_jacobi_lattice():
    size = (64, 40, 3)
    so = [(size, (a * size[0], b * size[1], c * size[2])) for c in range(2) for b in range(2) for a in range(2)]
    o, g = _pair(so, seed=12)
    want, hist = _run(o, g, "block_jacobi", steps=2)
    for po, pg in zip(o.patches, g.patches):
        assert G.rel_maxnorm(pg.u.cpu().numpy(), po.u) < TOL
    assert G.hist_rel(hist, want) < TOL


def test_band_and_dst_forms_agree():
    """Same level, same sweeps, the two device plane inverses (1e-13)."""
    shape = (256, 96, 4)
    rng = np.random.default_rng(1)
    u0, f = rng.standard_normal(shape), rng.standard_normal(shape)
    outs = []
    for mode in ("auto", "dst"):
        prev = ps.plane_solver(mode)
        try:
            p = ps.Patch(ps.PatchDims(*shape))
            p.interior[...] = torch.from_numpy(u0).cuda()
            p.f[...] = torch.from_numpy(f).cuda()
            lv = ps.Level([p])
            cfg = ps.SmootherConfig(scheme="block_jacobi", block_dims=(256, 96, 1), steps=3)
            _, hist = ps.smooth(lv, cfg, ps.InverseCache())
            outs.append((p.u.cpu().numpy(), hist))
        finally:
            ps.plane_solver(prev)
    assert G.rel_maxnorm(outs[0][0], outs[1][0]) < 1e-13
    assert G.hist_rel(outs[0][1], outs[1][1]) < 1e-13


def test_plane_solver_switch_validates():
    with pytest.raises(ValueError):
        ps.plane_solver("fft")
