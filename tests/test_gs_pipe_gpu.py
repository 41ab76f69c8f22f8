"""Parity of the plane-pipelined line GS kernel (psm_line_gs_pipe.cu: even nx
that splits into <= 32 lane chunks of <= 8 cells) with the CPU restatement of the reference's serial
(lexicographic) block GS, through the public API.

Wavefront ("colour-ordered") mode: iterates and histories within 1e-12
relative max-norm.  Chaotic mode: per-sweep residual factor within 2% of the
serial GS.  The shapes cover plane counts that are not multiples of the
8-plane CTA unit, single planes and rows, multi-patch lattices and
non-symmetric stencils."""

import numpy as np
import pytest
import torch

import golden_io as G
import paper_1208_1975_b200 as ps
from oracle import restate as R

pytestmark = pytest.mark.gpu
TOL = 1e-12


def _pair(shapes_origins, seed, center=6.0, faces=(-1.0,) * 6):
    rng = np.random.default_rng(seed)
    ops, gps = [], []
    for shape, origin in shapes_origins:
        u0 = rng.standard_normal(shape)
        f = rng.standard_normal(shape)
        o = R.OPatch(shape, origin)
        o.u[1:-1, 1:-1, 1:-1] = u0
        o.f[:] = f
        g = ps.Patch(ps.PatchDims(*shape), origin)
        g.interior[...] = torch.from_numpy(u0).cuda()
        g.f[...] = torch.from_numpy(f).cuda()
        ops.append(o)
        gps.append(g)
    return R.OLevel(ops), ps.Level(gps)


def _run(o, g, steps, omega=1.0, mode="wavefront", center=6.0, faces=(-1.0,) * 6):
    nx = g.patches[0].dims.nx
    want = R.smooth(o, "chaotic_block_gs", (nx, 1, 1), omega=omega, steps=steps, center=center, faces=faces,
                    exact_norm=False)
    cfg = ps.SmootherConfig(scheme="chaotic_block_gs", block_dims=(nx, 1, 1), omega=omega, steps=steps,
                            strategy=ps.ExecutionStrategy.device(gs_mode=mode),
                            stencil=ps.Stencil7(center, faces))
    _, hist = ps.smooth(g, cfg, ps.InverseCache())
    return want, hist


@pytest.mark.parametrize(
    "shape",
    [(32, 7, 3), (64, 5, 9), (128, 12, 17), (256, 9, 8), (256, 3, 19), (128, 1, 1), (32, 1, 20), (64, 16, 1),
     (128, 33, 8), (256, 40, 24)],
)
def test_wavefront_gs_matches_serial_restatement(shape):
    o, g = _pair([(shape, (0, 0, 0))], seed=sum(shape))
    want, hist = _run(o, g, steps=2)
    for po, pg in zip(o.patches, g.patches):
        assert G.rel_maxnorm(pg.u.cpu().numpy(), po.u) < TOL
    assert G.hist_rel(hist, want) < TOL


def test_wavefront_gs_nonsymmetric_stencil_and_omega():
    center, faces = 6.5, (-1.2, -0.8, -1.0, -1.1, -0.9, -1.05)
    o, g = _pair([((128, 10, 11), (0, 0, 0))], seed=3, center=center, faces=faces)
    want, hist = _run(o, g, steps=3, omega=0.7, center=center, faces=faces)
    assert G.rel_maxnorm(g.patches[0].u.cpu().numpy(), o.patches[0].u) < TOL
    assert G.hist_rel(hist, want) < TOL


def test_wavefront_gs_lattice_with_interfaces():
    size = (64, 6, 9)
    so = [(size, (a * size[0], b * size[1], c * size[2])) for c in range(3) for b in range(2) for a in range(2)]
    o, g = _pair(so, seed=11)
    want, hist = _run(o, g, steps=2)
    for po, pg in zip(o.patches, g.patches):
        assert G.rel_maxnorm(pg.u.cpu().numpy(), po.u) < TOL
    assert G.hist_rel(hist, want) < TOL


def test_wavefront_gs_mixed_line_lengths():
    """Patches of different nx (two pipelined groups, one launch each)."""
    so = [((64, 6, 10), (0, 0, 0)), ((128, 6, 10), (64, 0, 0)), ((32, 6, 10), (192, 0, 0))]
    rng = np.random.default_rng(5)
    ops, gps = [], []
    for shape, origin in so:
        u0, f = rng.standard_normal(shape), rng.standard_normal(shape)
        o = R.OPatch(shape, origin)
        o.u[1:-1, 1:-1, 1:-1] = u0
        o.f[:] = f
        p = ps.Patch(ps.PatchDims(*shape), origin)
        p.interior[...] = torch.from_numpy(u0).cuda()
        p.f[...] = torch.from_numpy(f).cuda()
        ops.append(o)
        gps.append(p)
    o, g = R.OLevel(ops), ps.Level(gps)
    want = []
    # each patch runs line blocks of its own nx: block (>= max nx, 1, 1) truncates per patch
    cfg = ps.SmootherConfig(scheme="chaotic_block_gs", block_dims=(128, 1, 1), steps=2,
                            strategy=ps.ExecutionStrategy.device(gs_mode="wavefront"))
    want = R.smooth(o, "chaotic_block_gs", (128, 1, 1), steps=2, exact_norm=False)
    _, hist = ps.smooth(g, cfg, ps.InverseCache())
    for po, pg in zip(o.patches, g.patches):
        assert G.rel_maxnorm(pg.u.cpu().numpy(), po.u) < TOL
    assert G.hist_rel(hist, want) < TOL


@pytest.mark.parametrize("shape", [(128, 64, 40), (256, 32, 24)])
def test_chaotic_gs_factor_within_two_percent_of_serial(shape):
    o, g = _pair([(shape, (0, 0, 0))], seed=9)
    want, hist = _run(o, g, steps=4, mode="chaotic")
    for s in range(1, len(want)):
        got_f, ref_f = hist[s] / hist[s - 1], want[s] / want[s - 1]
        assert abs(got_f - ref_f) / ref_f < 0.02, (s, got_f, ref_f)


@pytest.mark.parametrize(
    "shape",
    # nx = nl lanes x NC cells with nl < 32 or NC not a power of two
    [(72, 20, 15), (80, 17, 9), (88, 12, 10), (96, 9, 16), (12, 10, 8), (42, 7, 5), (150, 8, 9), (180, 6, 7),
     (210, 5, 8), (200, 4, 11), (2, 5, 4), (24, 1, 9)],
)
def test_wavefront_gs_general_line_lengths(shape):
    o, g = _pair([(shape, (0, 0, 0))], seed=7 + sum(shape))
    want, hist = _run(o, g, steps=2)
    assert G.rel_maxnorm(g.patches[0].u.cpu().numpy(), o.patches[0].u) < TOL
    assert G.hist_rel(hist, want) < TOL


def test_wavefront_gs_mixed_table2_like_level():
    """Patches of the paper's mixed sizes' line lengths (64..96), abutting
    along x with partial faces: one pipelined group per nx."""
    so = [((64, 8, 9), (0, 0, 0)), ((72, 9, 10), (64, 0, 0)), ((80, 10, 8), (136, 0, 0)),
          ((88, 8, 11), (216, 1, 0)), ((96, 11, 9), (304, 0, 0))]
    o, g = _pair(so, seed=13)
    want = R.smooth(o, "chaotic_block_gs", (96, 1, 1), steps=2, exact_norm=False)
    cfg = ps.SmootherConfig(scheme="chaotic_block_gs", block_dims=(96, 1, 1), steps=2,
                            strategy=ps.ExecutionStrategy.device(gs_mode="wavefront"))
    _, hist = ps.smooth(g, cfg, ps.InverseCache())
    for po, pg in zip(o.patches, g.patches):
        assert G.rel_maxnorm(pg.u.cpu().numpy(), po.u) < TOL
    assert G.hist_rel(hist, want) < TOL


def test_chaotic_gs_factor_general_line_length():
    o, g = _pair([((96, 48, 40), (0, 0, 0))], seed=21)
    want, hist = _run(o, g, steps=4, mode="chaotic")
    for s in range(1, len(want)):
        got_f, ref_f = hist[s] / hist[s - 1], want[s] / want[s - 1]
        assert abs(got_f - ref_f) / ref_f < 0.02, (s, got_f, ref_f)


# ---- multi-sweep mode (one launch runs every step of smooth(); single patch,
# physical faces): sweep s+1 trails sweep s inside the launch ----------------
@pytest.mark.parametrize("shape,steps", [((256, 24, 20), 5), ((128, 30, 7), 4), ((64, 9, 15), 6), ((72, 11, 8), 3),
                                         ((32, 1, 9), 3), ((64, 12, 1), 3), ((256, 5, 8), 2)])
def test_multisweep_wavefront_matches_serial(shape, steps):
    o, g = _pair([(shape, (0, 0, 0))], seed=40 + sum(shape))
    want, hist = _run(o, g, steps=steps)
    assert G.rel_maxnorm(g.patches[0].u.cpu().numpy(), o.patches[0].u) < TOL
    assert G.hist_rel(hist, want) < TOL


def test_multisweep_nonunit_stencil():
    center, faces = 6.5, (-1.2, -0.8, -1.0, -1.1, -0.9, -1.05)
    o, g = _pair([((128, 14, 16), (0, 0, 0))], seed=8, center=center, faces=faces)
    want, hist = _run(o, g, steps=4, omega=0.9, center=center, faces=faces)
    assert G.rel_maxnorm(g.patches[0].u.cpu().numpy(), o.patches[0].u) < TOL
    assert G.hist_rel(hist, want) < TOL


def test_multisweep_chaotic_factor():
    o, g = _pair([((256, 48, 40), (0, 0, 0))], seed=12)
    want, hist = _run(o, g, steps=8, mode="chaotic")
    for s in range(1, len(want)):
        got_f, ref_f = hist[s] / hist[s - 1], want[s] / want[s - 1]
        assert abs(got_f - ref_f) / ref_f < 0.02, (s, got_f, ref_f)


def test_multisweep_equals_step_by_step():
    """smooth() (graph, one multi-sweep launch) vs the eager per-step path
    (timers): identical iterates; histories to rounding (the in-kernel
    residual sums group the cells differently)."""
    shape = (128, 20, 18)
    a = _pair([(shape, (0, 0, 0))], seed=2)[1]
    b = _pair([(shape, (0, 0, 0))], seed=2)[1]
    cfg = ps.SmootherConfig(scheme="chaotic_block_gs", block_dims=(128, 1, 1), steps=6,
                            strategy=ps.ExecutionStrategy.device(gs_mode="wavefront"))
    _, ha = ps.smooth(a, cfg, ps.InverseCache())
    _, hb = ps.smooth(b, cfg, ps.InverseCache(), {})
    assert torch.equal(a.patches[0].u, b.patches[0].u)
    assert max(abs(x - y) / y for x, y in zip(ha, hb)) < 1e-14
