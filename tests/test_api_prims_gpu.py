"""The reference's per-block primitives on the device against the
reference's own outputs (tests/golden/api_prims.npz, made by
oracle/make_api_golden.py running patchsmooth): block_residual,
apply_stencil, matvec and block_update bit-identical; assemble_patch_matrix
exact; invert_dense within 1e-12 (multiply-back and entries);
spectral_radius_oracle within the power iteration's 1e-8 tolerance."""

import numpy as np
import pytest
import torch

import golden_io as G
import paper_1208_1975_b200 as ps

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def gold():
    return G.load("api_prims")


def _patch(d):
    p = ps.Patch(ps.PatchDims(*(int(n) for n in d["patch_shape"])))
    p.u.copy_(torch.from_numpy(d["patch_u"]))
    p.f.copy_(torch.from_numpy(d["patch_f"]))
    st = ps.Stencil7(float(d["stencil"][0]), tuple(float(c) for c in d["stencil"][1:]))
    return p, st


def test_block_residual_bitwise(gold):
    p, st = _patch(gold)
    for i in range(4):
        blk = ps.BlockRange(tuple(gold[f"block{i}_lo"]), tuple(gold[f"block{i}_ext"]))
        got = ps.block_residual(st, p, blk)
        assert got.is_cuda
        np.testing.assert_array_equal(got.cpu().numpy(), gold[f"block{i}_r"])


def test_block_residual_validation(gold):
    p, st = _patch(gold)
    with pytest.raises(ValueError):
        ps.block_residual(st, p, ps.BlockRange((5, 0, 0), (9, 1, 1)))
    with pytest.raises(TypeError):
        ps.block_residual(st, p, ((0, 0, 0), (1, 1, 1)))


def test_apply_stencil_bitwise(gold):
    p, st = _patch(gold)
    for c, want in zip(gold["apply_cells"], gold["apply_vals"]):
        assert ps.apply_stencil(st, p, tuple(int(v) for v in c)) == want
    with pytest.raises(ValueError):
        ps.apply_stencil(st, p, (9, 0, 0))


def test_assemble_patch_matrix_exact(gold):
    _, st = _patch(gold)
    got = ps.assemble_patch_matrix(st, ps.PatchDims(*(int(n) for n in gold["patch_matrix_dims"])))
    np.testing.assert_array_equal(got.cpu().numpy(), gold["patch_matrix"])


@pytest.mark.parametrize("n", [1, 7, 64, 200])
def test_matvec_and_block_update_bitwise(gold, n):
    m, x, u = gold[f"matvec{n}_m"], gold[f"matvec{n}_x"], gold[f"matvec{n}_u"]
    np.testing.assert_array_equal(ps.matvec(m, x), gold[f"matvec{n}_y"])  # numpy in, numpy out
    got = ps.matvec(torch.from_numpy(m).cuda(), torch.from_numpy(x).cuda())
    assert got.is_cuda
    np.testing.assert_array_equal(got.cpu().numpy(), gold[f"matvec{n}_y"])
    np.testing.assert_array_equal(ps.block_update(u, x, m, 0.7), gold[f"matvec{n}_upd"])


@pytest.mark.parametrize("n", [1, 5, 48])
def test_invert_dense(gold, n):
    a, want = gold[f"inv{n}_a"], gold[f"inv{n}_x"]
    got = ps.invert_dense(a)
    assert G.rel_maxnorm(got, want) < 1e-12
    assert ps.multiply_back_error(a, got) < 1e-12


def test_invert_dense_block_matrix(gold):
    got = ps.invert_dense(torch.from_numpy(gold["inv_blockmat"]).cuda())
    assert got.is_cuda
    assert G.rel_maxnorm(got.cpu().numpy(), gold["inv_blockmat_x"]) < 1e-13


def test_invert_dense_singular_and_bad_input():
    with pytest.raises(ps.SingularMatrixError):
        ps.invert_dense(np.zeros((3, 3)))
    with pytest.raises(ps.SingularMatrixError):
        ps.invert_dense(np.array([[1.0, 2.0], [2.0, 4.0]]))
    with pytest.raises(ValueError):
        ps.invert_dense(np.ones((2, 3)))
    with pytest.raises(ValueError):
        ps.invert_dense(np.array([[np.nan]]))


def test_spectral_radius_oracle(gold):
    for row in gold["rho_cases"]:
        dims, block = tuple(int(v) for v in row[:3]), tuple(int(v) for v in row[3:6])
        scheme = "chaotic_block_gs" if row[6] else "block_jacobi"
        r = ps.spectral_radius_oracle(ps.PatchDims(*dims), block, scheme)
        assert r.converged == bool(row[9])
        if r.converged:
            assert abs(r.rho - row[7]) < 1e-7 * row[7], (dims, block, r, row[7])
        else:
            assert r.iterations == 50000 and abs(r.rho - row[7]) < 0.05 * row[7]


def test_spectral_radius_oracle_anchors():
    """reference spectral radii of 8^3 line / plane blocks."""
    d = ps.PatchDims(8, 8, 8)
    assert abs(ps.spectral_radius_oracle(d, (8, 1, 1), "block_jacobi").rho - 0.911618881) < 1e-8
    assert abs(ps.spectral_radius_oracle(d, (8, 8, 1), "block_jacobi").rho - 0.839037027) < 1e-8
