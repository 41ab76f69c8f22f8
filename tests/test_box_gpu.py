"""Box blocks (the paper's cubic blocks, DEFAULT_BLOCK_SIZES 2^3..8^3): the
separable exact inverse (psm_box.cu) against the restatement's dense
inverses (the reference's invert_dense + matvec form) at sizes beyond the
golden fixtures (odd widths: cp.async staging; even widths: TMA staging;
a 240-block GS sweep through the ticket pipeline); Jacobi and lexicographic
GS iterates and histories within 1e-12; the explicit inverse equals the
dense one."""

import numpy as np
import pytest
import torch

import golden_io as G
import paper_1208_1975_b200 as ps
from oracle import restate as R

pytestmark = pytest.mark.gpu
TOL = 1e-12
SIZES = [(2, 2, 2), (4, 2, 2), (4, 4, 2), (4, 4, 4), (8, 4, 4), (8, 8, 4), (8, 8, 8)]  # analysis.py:38-46


def _pair(shape, seed):
    rng = np.random.default_rng(seed)
    u0, f = rng.standard_normal(shape), rng.standard_normal(shape)
    o = R.OPatch(shape)
    o.u[1:-1, 1:-1, 1:-1] = u0
    o.f[:] = f
    g = ps.Patch(ps.PatchDims(*shape))
    g.interior[...] = torch.from_numpy(u0).cuda()
    g.f[...] = torch.from_numpy(f).cuda()
    return R.OLevel([o]), ps.Level([g])


@pytest.mark.parametrize("block", SIZES)
@pytest.mark.parametrize("scheme", ["block_jacobi", "chaotic_block_gs"])
def test_default_block_sizes_match_dense_restatement(block, scheme):
    shape = (21, 18, 13)  # every axis truncates
    o, g = _pair(shape, seed=sum(block))
    want = R.smooth(o, scheme, block, steps=2, exact_norm=False)
    cfg = ps.SmootherConfig(scheme=scheme, block_dims=block, steps=2)
    _, hist = ps.smooth(g, cfg, ps.InverseCache())
    assert G.rel_maxnorm(g.patches[0].u.cpu().numpy(), o.patches[0].u) < TOL
    assert G.hist_rel(hist, want) < TOL


@pytest.mark.parametrize("block", SIZES)
@pytest.mark.parametrize("scheme", ["block_jacobi", "chaotic_block_gs"])
def test_default_block_sizes_even_width_tma_staging(block, scheme):
    """Even nx: 8^3 regions stage through TMA tensor copies (odd nx above
    takes the cp.async fallback); y and z still truncate."""
    shape = (24, 18, 14)
    o, g = _pair(shape, seed=3 + sum(block))
    want = R.smooth(o, scheme, block, steps=2, exact_norm=False)
    cfg = ps.SmootherConfig(scheme=scheme, block_dims=block, steps=2)
    _, hist = ps.smooth(g, cfg, ps.InverseCache())
    assert G.rel_maxnorm(g.patches[0].u.cpu().numpy(), o.patches[0].u) < TOL
    assert G.hist_rel(hist, want) < TOL


def test_box_gs_many_blocks_ticket_pipeline():
    """8^3 GS over 240 blocks (many CTAs, each holding two tickets, halos
    prefetched as soon as the predecessors are done): still exactly the
    lexicographic sweep."""
    o, g = _pair((64, 40, 48), seed=17)
    want = R.smooth(o, "chaotic_block_gs", (8, 8, 8), steps=2, exact_norm=False)
    cfg = ps.SmootherConfig(scheme="chaotic_block_gs", block_dims=(8, 8, 8), steps=2)
    _, hist = ps.smooth(g, cfg, ps.InverseCache())
    assert G.rel_maxnorm(g.patches[0].u.cpu().numpy(), o.patches[0].u) < TOL
    assert G.hist_rel(hist, want) < TOL


def test_box_nonsymmetric_faces_and_omega():
    center, faces = 7.2, (-1.3, -0.7, -1.1, -0.9, -0.8, -1.2)
    o, g = _pair((24, 16, 12), seed=9)
    want = R.smooth(o, "block_jacobi", (8, 4, 4), omega=0.65, steps=3, center=center, faces=faces,
                    exact_norm=False)
    cfg = ps.SmootherConfig(scheme="block_jacobi", block_dims=(8, 4, 4), omega=0.65, steps=3,
                            stencil=ps.Stencil7(center, faces))
    _, hist = ps.smooth(g, cfg, ps.InverseCache())
    assert G.rel_maxnorm(g.patches[0].u.cpu().numpy(), o.patches[0].u) < TOL
    assert G.hist_rel(hist, want) < TOL


@pytest.mark.parametrize("ext", [(8, 8, 8), (3, 5, 2), (8, 1, 1), (1, 1, 7)])
def test_box_explicit_inverse_equals_dense(ext):
    st = ps.Stencil7(6.5, (-1.2, -0.8, -1.0, -1.0, -0.9, -1.1))
    f = ps.BlockFactors(st, ext, "cuda")
    got = torch.linalg.inv(torch.eye(1, device="cuda"))  # warm cuBLAS/cuSOLVER-free path
    fh = f.handle_for("box")
    n = ext[0] * ext[1] * ext[2]
    eye = torch.eye(n, dtype=torch.float64, device="cuda")
    out = torch.empty_like(eye)
    import ctypes
    from paper_1208_1975_b200 import _lib
    _lib.check(_lib.load().psm_factors_apply(fh, ctypes.c_void_p(eye.data_ptr()), ctypes.c_void_p(out.data_ptr()),
                                             n, ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)))
    want = R.box_inverse(ext, st.center, st.faces)
    got = out.T.cpu().numpy()  # row j of out = Ainv e_j
    assert np.max(np.abs(got - want)) / np.max(np.abs(want)) < 1e-13


def test_box_opposite_sign_faces_are_rejected():
    with pytest.raises(ValueError):
        ps.BlockFactors(ps.Stencil7(6.0, (-1.0, 0.5, -1.0, -1.0, -1.0, -1.0)), (4, 4, 4), "cuda")
