"""Parity at the exact BASELINE.json configurations (C1, C2, C3, C4 and the
north-star 512^3 line-Jacobi grid), through the public API and so through
libpsmooth.so, against the CPU restatement of the reference:

* C1  64^3 single patch, line Jacobi over 10 sweeps (and two more small
  shapes) against the serial restatement;
* C2  256^3 single patch, line GS: wavefront ("colour-ordered") mode within
  1e-12 of the serial lexicographic sweep (iterates and history) over 2
  sweeps; chaotic mode's per-sweep residual factor within 2% of the serial
  sweep's over 10 sweeps;
* C3  512^3 single patch, plane Jacobi with exact plane inversion;
* C4  the 4x4x4 lattice of 128^3 patches (288 interface copies): line GS in
  both modes, plane GS, line and plane Jacobi;
* 512^3 line Jacobi (the north-star roofline grid).

Inputs follow SURVEY 8d: u0 from ``seed_initial_guess(level, 42)``, f
standard normal from ``default_rng(43)`` in patch order.  Line-block
references run on the C restatement (oracle/psm_oracle.c, pinned to the
reference's fixtures in test_oracle_golden.py), plane-block references on
the numpy restatement (oracle/restate.py)."""

import numpy as np
import pytest
import torch

import golden_io as G
import paper_1208_1975_b200 as ps
from oracle import cport
from oracle import restate as R

pytestmark = pytest.mark.gpu
TOL = 1e-12
FACTOR_TOL = 0.02


def _levels(counts, size):
    """The same level on the host (restatement) and on the device."""
    o = R.lattice_level(counts, size)
    g = ps.build_lattice(counts, size)
    rng_u, rng_f = np.random.default_rng(42), np.random.default_rng(43)
    for po, pg in zip(o.patches, g.patches):
        po.u[1:-1, 1:-1, 1:-1] = rng_u.random(po.dims)
        po.f[:] = rng_f.standard_normal(po.dims)
        pg.interior.copy_(torch.from_numpy(np.ascontiguousarray(po.u[1:-1, 1:-1, 1:-1])))
        pg.f.copy_(torch.from_numpy(np.ascontiguousarray(po.f)))
    return o, g


def _device_smooth(g, scheme, block, steps, mode="wavefront"):
    cfg = ps.SmootherConfig(scheme=scheme, block_dims=block, steps=steps,
                            strategy=ps.ExecutionStrategy.device(gs_mode=mode))
    _, hist = ps.smooth(g, cfg, ps.InverseCache())
    return hist


def _assert_iterates(o, g):
    worst = 0.0
    for po, pg in zip(o.patches, g.patches):
        worst = max(worst, G.rel_maxnorm(pg.u.cpu().numpy(), po.u))
    assert worst < TOL, worst


def _assert_factors(hist, want):
    for s in range(1, len(want)):
        got_f, ref_f = hist[s] / hist[s - 1], want[s] / want[s - 1]
        assert abs(got_f - ref_f) / ref_f < FACTOR_TOL, (s, got_f, ref_f)


# ---------------------------------------------------------------- C2
def test_c2_wavefront_line_gs_256():
    o, g = _levels((1, 1, 1), (256, 256, 256))
    want = cport.line_smooth(o, "chaotic_block_gs", steps=2)
    hist = _device_smooth(g, "chaotic_block_gs", (256, 1, 1), 2, "wavefront")
    _assert_iterates(o, g)
    assert G.hist_rel(hist, want) < TOL


def test_c2_chaotic_line_gs_256_ten_sweeps():
    o, g = _levels((1, 1, 1), (256, 256, 256))
    want = cport.line_smooth(o, "chaotic_block_gs", steps=10)
    hist = _device_smooth(g, "chaotic_block_gs", (256, 1, 1), 10, "chaotic")
    assert len(hist) == 11
    _assert_factors(hist, want)


# ---------------------------------------------------------------- C1
@pytest.mark.parametrize("shape,steps", [((64, 64, 64), 10), ((128, 64, 32), 3), ((64, 96, 40), 5)])
def test_c1_small_line_jacobi(shape, steps):
    """Small single-patch levels (the one-tile-per-CTA line kernel):
    iterates and every history entry against the serial restatement, odd
    and even sweep counts (final buffer parity)."""
    o, g = _levels((1, 1, 1), shape)
    want = cport.line_smooth(o, "block_jacobi", steps=steps)
    hist = _device_smooth(g, "block_jacobi", (shape[0], 1, 1), steps)
    assert len(hist) == steps + 1
    _assert_iterates(o, g)
    assert G.hist_rel(hist, want) < TOL


# ---------------------------------------------------------------- C3
def test_c3_plane_jacobi_512():
    o, g = _levels((1, 1, 1), (512, 512, 512))
    want = R.smooth(o, "block_jacobi", (512, 512, 1), steps=1, exact_norm=False)
    hist = _device_smooth(g, "block_jacobi", (512, 512, 1), 1)
    _assert_iterates(o, g)
    assert G.hist_rel(hist, want) < TOL


# ---------------------------------------------------------------- north star
def test_line_jacobi_512_two_sweeps():
    o, g = _levels((1, 1, 1), (512, 512, 512))
    want = cport.line_smooth(o, "block_jacobi", steps=2)
    hist = _device_smooth(g, "block_jacobi", (512, 1, 1), 2)
    _assert_iterates(o, g)
    assert G.hist_rel(hist, want) < TOL


# ---------------------------------------------------------------- C4
C4 = ((4, 4, 4), (128, 128, 128))


def test_c4_lattice_has_288_interface_copies():
    o = R.lattice_level(*C4)
    assert len(o.adjacency) == 288
    g = ps.build_lattice(*C4)
    assert len(g.adjacency) == 288


def test_c4_wavefront_line_gs():
    o, g = _levels(*C4)
    want = cport.line_smooth(o, "chaotic_block_gs", steps=2)
    hist = _device_smooth(g, "chaotic_block_gs", (128, 1, 1), 2, "wavefront")
    _assert_iterates(o, g)
    assert G.hist_rel(hist, want) < TOL


def test_c4_chaotic_line_gs_factor():
    o, g = _levels(*C4)
    want = cport.line_smooth(o, "chaotic_block_gs", steps=4)
    hist = _device_smooth(g, "chaotic_block_gs", (128, 1, 1), 4, "chaotic")
    _assert_factors(hist, want)


def test_c4_line_jacobi():
    o, g = _levels(*C4)
    want = cport.line_smooth(o, "block_jacobi", steps=2)
    hist = _device_smooth(g, "block_jacobi", (128, 1, 1), 2)
    _assert_iterates(o, g)
    assert G.hist_rel(hist, want) < TOL


def test_c4_plane_gs():
    o, g = _levels(*C4)
    want = R.smooth(o, "chaotic_block_gs", (128, 128, 1), steps=1, exact_norm=False)
    hist = _device_smooth(g, "chaotic_block_gs", (128, 128, 1), 1)
    _assert_iterates(o, g)
    assert G.hist_rel(hist, want) < TOL


def test_c4_plane_jacobi():
    o, g = _levels(*C4)
    want = R.smooth(o, "block_jacobi", (128, 128, 1), steps=1, exact_norm=False)
    hist = _device_smooth(g, "block_jacobi", (128, 128, 1), 1)
    _assert_iterates(o, g)
    assert G.hist_rel(hist, want) < TOL
