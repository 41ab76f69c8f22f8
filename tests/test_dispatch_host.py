"""for_each_patch_block (reference runtime.py:152-209) on the host: every
block exactly once under every strategy, lexicographic order for serial,
the first failure propagates, and decomposition-count validation
(reference test_runtime.py:43-57, :92-102)."""

import threading

import pytest
import torch

import paper_1208_1975_b200 as ps

CPU = torch.device("cpu")
STRATEGIES = [
    ps.ExecutionStrategy.serial(),
    ps.ExecutionStrategy.patch_parallel(3),
    ps.ExecutionStrategy.block_parallel(4),
    ps.ExecutionStrategy.two_level(2, 3),
    ps.ExecutionStrategy.device(),
]


def _level():
    lv = ps.build_level([(6, 4, 3), (3, 4, 3), (5, 4, 3)], device=CPU)
    decomps = [ps.decompose_blocks(p.dims, (2, 2, 2)) for p in lv.patches]
    return lv, decomps


@pytest.mark.parametrize("strategy", STRATEGIES, ids=lambda s: s.kind)
def test_every_block_exactly_once(strategy):
    lv, decomps = _level()
    seen, lock = [], threading.Lock()

    def work(pi, bi):
        with lock:
            seen.append((pi, bi))

    ps.for_each_patch_block(lv, decomps, strategy, work)
    want = [(pi, bi) for pi, d in enumerate(decomps) for bi in range(len(d.ranges))]
    assert sorted(seen) == want
    if strategy.kind in ("serial", "device"):
        assert seen == want


@pytest.mark.parametrize("strategy", STRATEGIES, ids=lambda s: s.kind)
def test_failure_propagates(strategy):
    lv, decomps = _level()

    def work(pi, bi):
        if (pi, bi) == (1, 2):
            raise KeyError("boom")

    with pytest.raises(KeyError):
        ps.for_each_patch_block(lv, decomps, strategy, work)


def test_decomposition_count_checked():
    lv, decomps = _level()
    with pytest.raises(ValueError):
        ps.for_each_patch_block(lv, decomps[:2], ps.ExecutionStrategy.serial(), lambda a, b: None)


def test_build_level_cap(monkeypatch):
    with pytest.raises(ValueError):
        ps.build_level([(64, 64, 64)], 1000, device=CPU)
    monkeypatch.setenv("PATCHSMOOTH_MAX_CELLS", "100")
    with pytest.raises(ValueError):
        ps.build_level([(8, 8, 8)], device=CPU)
    monkeypatch.setenv("PATCHSMOOTH_MAX_CELLS", "abc")
    with pytest.raises(ValueError):
        ps.build_level([(8, 8, 8)], device=CPU)
    monkeypatch.delenv("PATCHSMOOTH_MAX_CELLS")
    lv = ps.build_level([(4, 3, 2), (2, 3, 2)], None, CPU)
    assert [p.origin for p in lv.patches] == [(0, 0, 0), (4, 0, 0)]


def test_patch_set_specs():
    mixed = ps.PatchSetSpec.mixed_table2()
    assert mixed.count == 80 and len(mixed.sizes) == 80 and mixed.label == "mixed-table2"
    assert mixed.sizes[0] == (64, 64, 64) and mixed.sizes[-1] == (96, 96, 96)
    u = ps.PatchSetSpec.uniform((8, 4, 2), 3)
    assert u.sizes == [(8, 4, 2)] * 3 and u.label == "8x4x2-n3"
    assert ps.PatchSetSpec.uniform((8, 4, 2)).label == "8x4x2"
    for bad in (dict(kind="other"), dict(kind="uniform", size=(0, 1, 1)), dict(kind="uniform", size=(1, 1, 1), count=0)):
        with pytest.raises(ValueError):
            ps.PatchSetSpec(**bad)
