"""Parity of the CUDA path with the reference (golden fixtures made by running
patchsmooth itself) and with the CPU restatement at sizes the reference
cannot reach.  Everything here runs through the public package API, i.e.
through libpsmooth.so's C ABI.

Tolerances (north star): Jacobi and ordered GS iterates and histories within
1e-12 relative max-norm; chaotic GS per-sweep residual factor within 2%."""

import math

import numpy as np
import pytest
import torch

import golden_io as G
import paper_1208_1975_b200 as ps
from oracle import restate as R

pytestmark = pytest.mark.gpu
TOL = 1e-12


def _cfg(d, strategy=None, steps=None):
    st = ps.Stencil7(float(d["center"]), tuple(float(c) for c in d["faces"])) if "center" in d else ps.Stencil7()
    return ps.SmootherConfig(
        scheme=str(d["scheme"]),
        block_dims=tuple(int(b) for b in d["block"]),
        omega=float(d["omega"]),
        steps=int(d["steps"]) if steps is None else steps,
        strategy=strategy if strategy is not None else ps.ExecutionStrategy.serial(),
        stencil=st,
    )


def _np(t):
    return t.detach().cpu().numpy()


def _single_level(d):
    p = ps.Patch(ps.PatchDims(*(int(n) for n in d["shape"])))
    p.interior[...] = torch.from_numpy(d["u0"]).cuda()
    p.f[...] = torch.from_numpy(d["f"]).cuda()
    return ps.Level([p])


@pytest.mark.parametrize("name", G.single_patch_cases())
def test_single_patch_matches_reference(name):
    d = G.load(name)
    lv = _single_level(d)
    _, hist = ps.smooth(lv, _cfg(d), ps.InverseCache())
    u = _np(lv.patches[0].u)
    assert G.rel_maxnorm(u[1:-1, 1:-1, 1:-1], d["u_final"][1:-1, 1:-1, 1:-1]) < TOL
    assert G.rel_maxnorm(u, d["u_final"]) < TOL  # ghosts included
    if d["history"][0] > 0:
        assert G.hist_rel(hist, d["history"]) < TOL


@pytest.mark.parametrize("name", G.multipatch_cases())
def test_multipatch_matches_reference(name):
    d = G.load(name)
    lv = ps.build_lattice(tuple(int(c) for c in d["counts"]), tuple(int(s) for s in d["size"]))
    for p, u0, f in zip(lv.patches, d["u0"], d["f"]):
        p.interior[...] = torch.from_numpy(u0).cuda()
        p.f[...] = torch.from_numpy(f).cuda()
    _, hist = ps.smooth(lv, _cfg(d), ps.InverseCache())
    for p, want in zip(lv.patches, d["u_final"]):
        assert G.rel_maxnorm(_np(p.u), want) < TOL
    assert G.hist_rel(hist, d["history"]) < TOL


@pytest.mark.parametrize("name", G.zsplit_cases())
def test_zsplit_matches_reference(name):
    d = G.load(name)
    nx, ny, nz = (int(n) for n in d["shape"])
    parts = int(d["parts"])
    dz = nz // parts
    lv = ps.Level([ps.Patch(ps.PatchDims(nx, ny, dz), (0, 0, g * dz)) for g in range(parts)])
    for g, p in enumerate(lv.patches):
        p.interior[...] = torch.from_numpy(np.ascontiguousarray(d["u0"][:, :, g * dz:(g + 1) * dz])).cuda()
        p.f[...] = torch.from_numpy(np.ascontiguousarray(d["f"][:, :, g * dz:(g + 1) * dz])).cuda()
    _, hist = ps.smooth(lv, _cfg(d), ps.InverseCache())
    got = np.concatenate([_np(p.interior) for p in lv.patches], axis=2)
    assert G.rel_maxnorm(got, d["interior_final"]) < TOL
    assert G.hist_rel(hist, d["history"]) < TOL


@pytest.mark.parametrize("name", ["seeded_line_jac_64", "seeded_line_gs_32", "seeded_plane_jac_32"])
def test_cli_inputs_match_reference(name):
    d = G.load(name)
    lv = ps.build_level([tuple(int(n) for n in d["shape"])])
    ps.seed_initial_guess(lv, 42)
    _, hist = ps.smooth(lv, _cfg(d), ps.InverseCache())
    assert G.hist_rel(hist, d["history"]) < TOL
    inter = _np(lv.patches[0].interior)
    for k, plane in zip(d["planes"], d["plane_values"]):
        assert G.rel_maxnorm(inter[:, :, int(k)], plane) < TOL


def test_chaotic_gs_factor_within_two_percent():
    """Chaotic mode vs the reference's serial GS, per-sweep factor (8 sweeps)."""
    d = G.load("seeded_line_gs_32")
    lv = ps.build_level([tuple(int(n) for n in d["shape"])])
    ps.seed_initial_guess(lv, 42)
    cfg = _cfg(d, strategy=ps.ExecutionStrategy.block_parallel(8))
    _, hist = ps.smooth(lv, cfg, ps.InverseCache())
    want = d["history"]
    for s in range(1, len(want)):
        got_f = hist[s] / hist[s - 1]
        ref_f = want[s] / want[s - 1]
        assert abs(got_f - ref_f) / ref_f < 0.02, (s, got_f, ref_f)


def test_refresh_and_norms_match_reference_bitwise():
    d = G.load("host_logic")
    dims = [(4, 4, 4), (4, 2, 4), (4, 2, 4), (3, 4, 2)]
    origins = [(0, 0, 0), (4, 0, 0), (4, 2, 0), (1, 0, 4)]
    lv = ps.Level([ps.Patch(ps.PatchDims(*s), o) for s, o in zip(dims, origins)])
    for i, p in enumerate(lv.patches):
        p.u[...] = torch.from_numpy(d[f"refresh_before_{i}"]).cuda()
    lv.refresh_ghosts()
    for i, p in enumerate(lv.patches):
        np.testing.assert_array_equal(_np(p.u), d[f"refresh_after_{i}"])
    assert ps.residual_norm(lv, ps.Stencil7()) == pytest.approx(float(d["norm_f_zero"]), rel=1e-14)
    for i, p in enumerate(lv.patches):
        p.f[...] = torch.from_numpy(d[f"norm_f_{i}"]).cuda()
    assert ps.residual_norm(lv, ps.Stencil7()) == pytest.approx(float(d["norm_with_f"]), rel=1e-14)


def _restated_level(shape, seed=7):
    rng = np.random.default_rng(seed)
    u0 = rng.standard_normal(shape)
    f = rng.standard_normal(shape)
    o = R.OPatch(shape)
    o.u[1:-1, 1:-1, 1:-1] = u0
    o.f[:] = f
    g = ps.Patch(ps.PatchDims(*shape))
    g.interior[...] = torch.from_numpy(u0).cuda()
    g.f[...] = torch.from_numpy(f).cuda()
    return R.OLevel([o]), ps.Level([g])


@pytest.mark.parametrize(
    "shape,scheme,block,steps",
    [
        ((256, 256, 256), "block_jacobi", (256, 1, 1), 2),
        ((256, 64, 48), "chaotic_block_gs", (256, 1, 1), 2),
        ((1024, 32, 16), "block_jacobi", (1024, 1, 1), 2),
        ((1000, 9, 7), "block_jacobi", (1000, 1, 1), 2),
        ((4096, 4, 3), "block_jacobi", (4096, 1, 1), 1),
        ((96, 40, 24), "chaotic_block_gs", (96, 1, 1), 2),
        ((600, 5, 4), "chaotic_block_gs", (600, 1, 1), 1),
        ((128, 128, 16), "block_jacobi", (128, 128, 1), 2),
        ((64, 48, 12), "chaotic_block_gs", (64, 64, 1), 2),
    ],
)
def test_large_sizes_match_restatement(shape, scheme, block, steps):
    o, g = _restated_level(shape)
    want = R.smooth(o, scheme, block, steps=steps, exact_norm=False)
    cfg = ps.SmootherConfig(scheme=scheme, block_dims=block, steps=steps)
    _, hist = ps.smooth(g, cfg, ps.InverseCache())
    assert G.rel_maxnorm(_np(g.patches[0].interior), o.patches[0].interior) < TOL
    assert G.hist_rel(hist, want) < TOL


def test_512_line_jacobi_matches_restatement():
    """North-star size, one sweep, against the CPU restatement."""
    o, g = _restated_level((512, 512, 512), seed=5)
    want = R.smooth(o, "block_jacobi", (512, 1, 1), steps=1, exact_norm=False)
    _, hist = ps.smooth(g, ps.SmootherConfig(scheme="block_jacobi", block_dims=(512, 1, 1)), ps.InverseCache())
    assert G.rel_maxnorm(_np(g.patches[0].interior), o.patches[0].interior) < TOL
    assert G.hist_rel(hist, want) < TOL


@pytest.mark.parametrize("scheme", ["block_jacobi", "chaotic_block_gs"])
@pytest.mark.parametrize("block", [(64, 1, 1), (64, 64, 1)])
def test_zero_field_is_a_fixed_point(scheme, block):
    lv = ps.Level([ps.Patch(ps.PatchDims(64, 20, 8))])
    _, hist = ps.smooth(lv, ps.SmootherConfig(scheme=scheme, block_dims=block, steps=3), ps.InverseCache())
    assert hist == [0.0, 0.0, 0.0, 0.0]
    assert float(lv.patches[0].u.abs().max()) == 0.0


@pytest.mark.parametrize("scheme", ["block_jacobi", "chaotic_block_gs"])
def test_exact_solution_is_a_fixed_point(scheme):
    """f = A u with the ghost rule folded in (reference test_smoother.py:113-128)."""
    shape = (96, 12, 10)
    rng = np.random.default_rng(3)
    o = R.OPatch(shape)
    o.u[1:-1, 1:-1, 1:-1] = rng.standard_normal(shape)
    R.fill_physical_ghosts(o.u)
    o.f[:] = R.residual(o.u, np.zeros(shape)) * -1.0  # A u
    p = ps.Patch(ps.PatchDims(*shape))
    p.interior[...] = torch.from_numpy(o.interior.copy()).cuda()
    p.f[...] = torch.from_numpy(o.f).cuda()
    before = _np(p.interior).copy()
    _, hist = ps.smooth(ps.Level([p]), ps.SmootherConfig(scheme=scheme, block_dims=(96, 1, 1), steps=2),
                        ps.InverseCache())
    np.testing.assert_allclose(_np(p.interior), before, rtol=0, atol=1e-12)
    assert all(h < 1e-10 for h in hist)


def _two_patch(seed):
    dims = ps.PatchDims(32, 8, 8)
    a, b = ps.Patch(dims), ps.Patch(dims, origin=(32, 0, 0))
    rng = np.random.default_rng(seed)
    for p in (a, b):
        p.interior[...] = torch.from_numpy(rng.standard_normal(dims.shape)).cuda()
        p.f[...] = torch.from_numpy(rng.standard_normal(dims.shape)).cuda()
    return ps.Level([a, b])


def test_jacobi_is_bitwise_invariant_across_strategies():
    S = ps.ExecutionStrategy
    results = []
    for strat in (S.serial(), S.patch_parallel(3), S.block_parallel(4), S.two_level(2, 2), S.device()):
        lv = _two_patch(21)
        cfg = ps.SmootherConfig(scheme="block_jacobi", block_dims=(32, 1, 1), steps=3, strategy=strat)
        _, hist = ps.smooth(lv, cfg, ps.InverseCache())
        results.append((hist, [_np(p.u) for p in lv.patches]))
    for hist, fields in results[1:]:
        assert hist == results[0][0]
        for a, b in zip(fields, results[0][1]):
            np.testing.assert_array_equal(a, b)


def test_jacobi_is_bitwise_invariant_under_zsplit():
    """The basis of multi-GPU z-slab parity: splitting one patch
    into z-slabs changes neither iterates nor history, bit for bit."""
    shape = (64, 16, 16)
    rng = np.random.default_rng(4)
    u0 = rng.standard_normal(shape)
    f = rng.standard_normal(shape)
    whole = ps.Level([ps.Patch(ps.PatchDims(*shape))])
    whole.patches[0].interior[...] = torch.from_numpy(u0).cuda()
    whole.patches[0].f[...] = torch.from_numpy(f).cuda()
    slabs = ps.Level([ps.Patch(ps.PatchDims(64, 16, 4), (0, 0, 4 * g)) for g in range(4)])
    for g, p in enumerate(slabs.patches):
        p.interior[...] = torch.from_numpy(np.ascontiguousarray(u0[:, :, 4 * g:4 * g + 4])).cuda()
        p.f[...] = torch.from_numpy(np.ascontiguousarray(f[:, :, 4 * g:4 * g + 4])).cuda()
    cfg = ps.SmootherConfig(scheme="block_jacobi", block_dims=(64, 1, 1), steps=4)
    _, h1 = ps.smooth(whole, cfg, ps.InverseCache())
    _, h2 = ps.smooth(slabs, cfg, ps.InverseCache())
    assert h1 == h2
    merged = np.concatenate([_np(p.interior) for p in slabs.patches], axis=2)
    np.testing.assert_array_equal(_np(whole.patches[0].interior), merged)


def test_step_functions_check_the_scheme_and_timers():
    lv = _two_patch(1)
    jac = ps.SmootherConfig(scheme="block_jacobi", block_dims=(32, 1, 1))
    gs = ps.SmootherConfig(scheme="chaotic_block_gs", block_dims=(32, 1, 1))
    with pytest.raises(ValueError):
        ps.smooth_jacobi_step(lv, gs, ps.InverseCache())
    with pytest.raises(ValueError):
        ps.smooth_chaotic_gs_step(lv, jac, ps.InverseCache())
    timers = {}
    ps.smooth(lv, ps.SmootherConfig(scheme="block_jacobi", block_dims=(32, 1, 1), steps=2), ps.InverseCache(),
              timers=timers)
    assert set(timers) == {"ghost_seconds"} and timers["ghost_seconds"] > 0.0


def test_single_steps_equal_smooth():
    a, b = _two_patch(9), _two_patch(9)
    cfg = ps.SmootherConfig(scheme="chaotic_block_gs", block_dims=(32, 1, 1), steps=2)
    ps.smooth(a, cfg, ps.InverseCache())
    b.refresh_ghosts()
    cache = ps.InverseCache()
    for _ in range(2):
        ps.smooth_chaotic_gs_step(b, cfg, cache)
    for p, q in zip(a.patches, b.patches):
        np.testing.assert_array_equal(_np(p.u), _np(q.u))


@pytest.mark.parametrize("extent", [(16, 1, 1), (37, 1, 1), (8, 6, 1), (12, 12, 1)])
def test_block_inverse_matches_dense(extent):
    """BlockFactors.dense() equals the inverse of the closure-free block
    operator (stencil.py:115-138) to rounding."""
    fac = ps.InverseCache().get(ps.Stencil7(), extent)
    inv = _np(fac.dense())
    ex, ey, _ = extent
    n = ex * ey
    a = np.zeros((n, n))
    for y in range(ey):
        for x in range(ex):
            r = x + ex * y
            a[r, r] = 6.0
            for dx, dy in ((-1, 0), (1, 0), (0, -1), (0, 1)):
                if 0 <= x + dx < ex and 0 <= y + dy < ey:
                    a[r, (x + dx) + ex * (y + dy)] = -1.0
    assert np.max(np.abs(a @ inv - np.eye(n))) < 1e-13


def test_inverse_cache_counts_and_binding():
    cache = ps.InverseCache()
    lv = _two_patch(2)
    cfg = ps.SmootherConfig(scheme="block_jacobi", block_dims=(32, 1, 1), steps=1)
    ps.smooth(lv, cfg, cache)
    ps.smooth(lv, cfg, cache)
    assert cache.inversions == 1 and cache.shapes == ((32, 1, 1),)
    with pytest.raises(ValueError):
        cache.get(ps.Stencil7(center=7.0), (32, 1, 1))


def test_weak_diagonal_dominance_uses_generic_kernel():
    """A stencil whose line inverse decays slowly (center 2.2) cannot use the
    32-segment partition; the plan falls back to the full-Thomas kernels."""
    st = ps.Stencil7(center=2.2, faces=(-1.0, -1.0, -0.05, -0.05, -0.05, -0.05))
    shape = (200, 6, 5)
    rng = np.random.default_rng(11)
    o = R.OPatch(shape)
    o.u[1:-1, 1:-1, 1:-1] = rng.standard_normal(shape)
    o.f[:] = rng.standard_normal(shape)
    p = ps.Patch(ps.PatchDims(*shape))
    p.interior[...] = torch.from_numpy(o.interior.copy()).cuda()
    p.f[...] = torch.from_numpy(o.f).cuda()
    for scheme in ("block_jacobi", "chaotic_block_gs"):
        want = R.smooth(R.OLevel([o]), scheme, (200, 1, 1), steps=2, center=st.center, faces=st.faces)
        _, hist = ps.smooth(ps.Level([p]), ps.SmootherConfig(scheme=scheme, block_dims=(200, 1, 1), steps=2,
                                                             stencil=st), ps.InverseCache())
        assert G.rel_maxnorm(_np(p.interior), o.interior) < 1e-11
        assert G.hist_rel(hist, want) < 1e-11


def test_north_star_array_form():
    shape = (64, 16, 12)
    rng = np.random.default_rng(2)
    u = rng.standard_normal(shape)
    f = rng.standard_normal(shape)
    o = R.OPatch(shape)
    o.u[1:-1, 1:-1, 1:-1] = u
    o.f[:] = f
    want = R.smooth(R.OLevel([o]), "chaotic_block_gs", (64, 64, 1), steps=3, exact_norm=False)
    ut = torch.from_numpy(u.copy()).cuda()
    out, hist = ps.smooth(ut, torch.from_numpy(f).cuda(), 3, block="plane", method="gs")
    assert out is ut
    assert G.rel_maxnorm(_np(ut), o.interior) < TOL
    assert G.hist_rel(hist, want) < TOL


def test_singular_and_unsupported_inputs_raise():
    with pytest.raises(ps.SingularMatrixError):
        ps.InverseCache().get(ps.Stencil7(center=1.0), (16, 1, 1))
    with pytest.raises(ValueError):
        ps.InverseCache().get(ps.Stencil7(faces=(-1.0, -0.5, -1.0, -1.0, -1.0, -1.0)), (8, 8, 1))
    lv = _two_patch(3)
    with pytest.raises(ValueError):
        ps.smooth(lv, ps.SmootherConfig(scheme="block_jacobi", block_dims=(16, 16, 16)), ps.InverseCache())
    assert math.isfinite(ps.residual_norm(lv, ps.Stencil7()))
