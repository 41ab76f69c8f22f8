"""The box sweep's fragment-register line orders (psm_box.cu box_jx / box_ip,
the two-shuffle register exchanges, the padded work cube) compute the
separable transform exactly and keep every shared-memory access
bank-conflict free: a lane-by-lane numpy simulation (tools/box_lanes_sim.py),
no GPU needed."""

import importlib.util
import os

import pytest

_SIM = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tools", "box_lanes_sim.py")


def _load():
    spec = importlib.util.spec_from_file_location("box_lanes_sim", _SIM)
    mod = importlib.util.module_from_spec(spec)
    spec.loader.exec_module(mod)
    return mod


@pytest.mark.parametrize("seed", [0, 1, 2])
def test_lane_orders_compute_the_separable_transform(seed):
    err, _ = _load().simulate(seed)
    assert err < 1e-14  # rounding only: the same products, another summation order


def test_shared_memory_accesses_are_conflict_free():
    _, issues = _load().simulate(0)
    assert issues == []
