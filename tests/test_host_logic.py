"""CPU-only checks of the package's host-side logic (no kernels run):
adjacency derivation against the reference's answers, config/strategy
validation, decomposition, block classification, patch partitioning."""

import numpy as np
import pytest
import torch

import golden_io as G
import paper_1208_1975_b200 as ps

CPU = torch.device("cpu")


def _adj(level):
    return [(c.src, c.dst, *c.src_lo, *c.dst_lo, *c.extent) for c in level.adjacency]


def _rows(a):
    return [tuple(int(v) for v in r) for r in a]


def test_build_level_adjacency_matches_reference():
    d = G.load("host_logic")
    lv = ps.build_level([(4, 3, 2), (2, 3, 2), (3, 3, 2)], device=CPU)
    assert _adj(lv) == _rows(d["build_level_adj"])


def test_partial_face_adjacency_matches_reference():
    d = G.load("host_logic")
    dims = [(4, 4, 4), (4, 2, 4), (4, 2, 4), (3, 4, 2)]
    origins = [(0, 0, 0), (4, 0, 0), (4, 2, 0), (1, 0, 4)]
    lv = ps.Level([ps.Patch(ps.PatchDims(*s), o, device=CPU) for s, o in zip(dims, origins)])
    assert _adj(lv) == _rows(d["partial_adj"])


def test_lattice_adjacency_matches_reference():
    d = G.load("host_logic")
    lv = ps.build_lattice((3, 2, 2), (3, 2, 4), device=CPU)
    assert _adj(lv) == _rows(d["lattice_adj"])


@pytest.mark.parametrize("name", G.multipatch_cases())
def test_multipatch_adjacency_matches_reference(name):
    d = G.load(name)
    lv = ps.build_lattice(tuple(int(c) for c in d["counts"]), tuple(int(s) for s in d["size"]), device=CPU)
    assert _adj(lv) == _rows(d["adjacency"])


def test_explicit_adjacency_is_validated():
    a = ps.Patch(ps.PatchDims(4, 4, 4), device=CPU)
    b = ps.Patch(ps.PatchDims(4, 4, 4), origin=(4, 0, 0), device=CPU)
    auto = ps.Level([a, b]).adjacency
    ps.Level([a, b], adjacency=auto)  # consistent and symmetric
    with pytest.raises(ValueError):
        ps.Level([a, b], adjacency=auto[:1])  # missing mirror
    with pytest.raises(ValueError):
        ps.Level([a, ps.Patch(ps.PatchDims(4, 4, 4), origin=(2, 0, 0), device=CPU)])  # overlap


def test_patch_layout_matches_reference_memory_order():
    p = ps.Patch(ps.PatchDims(5, 4, 3), device=CPU)
    assert tuple(p.u.shape) == (7, 6, 5)
    assert tuple(p.f.shape) == (5, 4, 3)
    # x fastest: stride 1 along i, padded row along j, padded plane along k
    assert p.u.stride() == (1, 7, 42)
    assert p.f.stride() == (1, 5, 20)
    assert ps.global_index(p.dims, (0, 0, 0), with_ghost=True) == 1 + 7 + 42
    p.u[2, 3, 1] = 9.0
    flat = p._bufs[0].reshape(-1)
    assert flat[ps.global_index(p.dims, (1, 2, 0), with_ghost=True)] == 9.0


def test_patch_f_assignment_keeps_storage():
    p = ps.Patch(ps.PatchDims(3, 2, 2), device=CPU)
    ptr = p._f.data_ptr()
    p.f = np.arange(12.0).reshape(3, 2, 2)
    assert p._f.data_ptr() == ptr
    assert float(p.f[2, 1, 1]) == 11.0


def test_swap_buffers_is_a_role_flip():
    p = ps.Patch(ps.PatchDims(2, 2, 2), device=CPU)
    p.u[1, 1, 1] = 3.0
    p.swap_buffers()
    assert float(p.u[1, 1, 1]) == 0.0
    assert float(p.v[0, 0, 0]) == 3.0
    p.swap_buffers()
    assert float(p.interior[0, 0, 0]) == 3.0


def test_decompose_blocks_truncation():
    dec = ps.decompose_blocks(ps.PatchDims(5, 4, 3), (2, 4, 2))
    assert dec.counts == (3, 1, 2)
    assert dec.ranges[2].extent == (1, 4, 2)
    assert dec.shapes == ((2, 4, 2), (1, 4, 2), (2, 4, 1), (1, 4, 1))
    assert dec.block_of((4, 3, 2)) == 5


@pytest.mark.parametrize(
    "dims,block,want",
    [
        ((64, 8, 8), (64, 1, 1), ((64, 1, 1), "line")),
        ((64, 8, 8), (128, 1, 1), ((64, 1, 1), "line")),
        ((16, 16, 4), (16, 16, 1), ((16, 16, 1), "plane")),
        ((16, 16, 4), (32, 32, 1), ((16, 16, 1), "plane")),
        ((16, 1, 4), (16, 16, 1), ((16, 1, 1), "line")),
        ((64, 16, 8), (8, 8, 8), ((8, 8, 8), "box")),
        ((64, 16, 8), (4, 2, 2), ((4, 2, 2), "box")),
        ((6, 5, 3), (8, 8, 8), ((6, 5, 3), "box")),
        ((64, 16, 8), (8, 1, 1), ((8, 1, 1), "box")),
    ],
)
def test_block_shape_classification(dims, block, want):
    assert ps.block_shape_of(ps.PatchDims(*dims), block) == want


@pytest.mark.parametrize("block", [(16, 16, 16), (32, 1, 1), (64, 2, 1), (64, 8, 2), (9, 2, 2)])
def test_unsupported_blocks_are_rejected(block):
    with pytest.raises(ValueError):
        ps.block_shape_of(ps.PatchDims(64, 16, 8), block)


def test_config_defaults_and_validation():
    # same contract as reference test_smoother.py:273-289
    assert ps.SmootherConfig(scheme="block_jacobi", block_dims=(2, 2, 2)).omega == 0.8
    assert ps.SmootherConfig(scheme="chaotic_block_gs", block_dims=(2, 2, 2)).omega == 1.0
    with pytest.raises(ValueError):
        ps.SmootherConfig(scheme="sor", block_dims=(2, 2, 2))
    with pytest.raises(ValueError):
        ps.SmootherConfig(scheme="block_jacobi", block_dims=(0, 2, 2))
    with pytest.raises(ValueError):
        ps.SmootherConfig(scheme="block_jacobi", block_dims=(2, 2, 2), omega=0.0)
    with pytest.raises(ValueError):
        ps.SmootherConfig(scheme="block_jacobi", block_dims=(2, 2, 2), omega=1.5)
    with pytest.raises(ValueError):
        ps.SmootherConfig(scheme="block_jacobi", block_dims=(2, 2, 2), steps=0)
    with pytest.raises(ValueError):
        ps.SmootherConfig(scheme="block_jacobi", block_dims=(2, 2, 2), seed=1.5)
    with pytest.raises(TypeError):
        ps.SmootherConfig(scheme="block_jacobi", block_dims=(2, 2, 2), strategy="serial")


def test_strategy_gs_modes():
    S = ps.ExecutionStrategy
    assert S.serial().resolved_gs_mode == "wavefront"
    assert S.patch_parallel(4).resolved_gs_mode == "wavefront"
    assert S.block_parallel(8).resolved_gs_mode == "chaotic"
    assert S.two_level(2, 2).resolved_gs_mode == "chaotic"
    assert S.device(gs_mode="chaotic").resolved_gs_mode == "chaotic"
    assert S.device(devices=8).width == 8
    with pytest.raises(ValueError):
        S(kind="device", gs_mode="redblack")
    with pytest.raises(ValueError):
        S(kind="gpu")


def test_partition_patches_matches_reference_rules():
    lv = ps.build_level([(8, 4, 4), (2, 4, 4), (6, 4, 4), (4, 4, 4)], device=CPU)
    assert ps.partition_patches(lv, 2, "greedy") == [[0, 1], [2, 3]]
    assert ps.partition_patches(lv, 3, "round_robin") == [[0, 3], [1], [2]]
    assert ps.partition_patches(lv, 3, "in_order") == [[0, 1], [2], [3]]


def test_smoothing_refuses_cpu_levels():
    lv = ps.build_level([(4, 4, 4)], device=CPU)
    cfg = ps.SmootherConfig(scheme="block_jacobi", block_dims=(4, 1, 1))
    with pytest.raises(RuntimeError):
        ps.smooth(lv, cfg, ps.InverseCache())


def test_ghost_overhead_paper_values():
    assert ps.ghost_overhead(ps.PatchDims(32, 32, 32))[0] == 6536
    assert ps.ghost_overhead(ps.PatchDims(64, 64, 64))[0] == 25352
