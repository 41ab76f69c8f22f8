"""The graph-replayed step sequence (psm_smooth_steps) equals the eager one
bitwise, for every scheme and block kind, across repeated calls (eager
first call, capture on the second, replay after), odd and even step counts,
and after the history workspace grows (graphs re-captured)."""

import numpy as np
import pytest
import torch

import paper_1208_1975_b200 as ps

pytestmark = pytest.mark.gpu


def _level(shape, seed, npatch=1):
    g = torch.Generator(device="cuda")
    g.manual_seed(seed)
    pts = []
    for i in range(npatch):
        p = ps.Patch(ps.PatchDims(*shape), origin=(i * shape[0], 0, 0))
        p.interior.copy_(torch.rand(p.interior.shape, dtype=torch.float64, device="cuda", generator=g))
        p.f.copy_(torch.randn(p.f.shape, dtype=torch.float64, device="cuda", generator=g))
        pts.append(p)
    return ps.Level(pts)


@pytest.mark.parametrize("scheme,block,steps,npatch", [
    ("block_jacobi", "line", 3, 1), ("block_jacobi", "line", 4, 2), ("chaotic_block_gs", "line", 3, 2),
    ("block_jacobi", "plane", 3, 1), ("chaotic_block_gs", "plane", 2, 2)])
def test_graph_replay_matches_eager(scheme, block, steps, npatch):
    shape = (64, 24, 10)
    bd = (64, 1, 1) if block == "line" else (64, 24, 1)
    cfg = ps.SmootherConfig(scheme=scheme, block_dims=bd, steps=steps)
    cache = ps.InverseCache()
    eager = _level(shape, 3, npatch)
    timers = {}
    _, h_eager = ps.smooth(eager, cfg, cache, timers)  # timers -> eager path
    lv = _level(shape, 3, npatch)
    hs = []
    for rep in range(4):  # eager, capture+replay, replay, replay
        for p, q in zip(lv.patches, _level(shape, 3, npatch).patches):
            p.u.copy_(q.u)
            p.f.copy_(q.f)
        _, h = ps.smooth(lv, cfg, cache)
        hs.append(h)
        for p, q in zip(lv.patches, eager.patches):
            assert torch.equal(p.u, q.u), rep
    for h in hs:
        assert h == h_eager


def test_graph_survives_history_growth():
    cfg2 = ps.SmootherConfig(scheme="block_jacobi", block_dims=(32, 1, 1), steps=2)
    cfg9 = ps.SmootherConfig(scheme="block_jacobi", block_dims=(32, 1, 1), steps=9)
    cache = ps.InverseCache()
    lv = _level((32, 16, 8), 5)
    ref = _level((32, 16, 8), 5)
    for _ in range(3):
        ps.smooth(lv, cfg2, cache)
        ps.smooth(ref, cfg2, cache, {})
    ps.smooth(lv, cfg9, cache)
    ps.smooth(ref, cfg9, cache, {})
    _, h = ps.smooth(lv, cfg2, cache)
    _, hr = ps.smooth(ref, cfg2, cache, {})
    assert h == hr
    assert torch.equal(lv.patches[0].u, ref.patches[0].u)
