"""Argument parsing of the device CLI (no GPU): the reference's validation
rules and exit status 2, plus the device flags."""

import pytest

from paper_1208_1975_b200 import cli


@pytest.mark.parametrize("argv", [
    ["smooth", "--steps", "0"], ["smooth", "--omega", "1.5"], ["smooth", "--patch-size", "4x4"],
    ["converge", "--num-patches", "2"], ["smooth", "--mixed-table2", "--num-patches", "2"],
    ["bench", "--patch-workers", "2"], ["smooth", "--devices", "2"], ["smooth", "--gs-mode", "chaotic"],
])
def test_bad_arguments_exit_2(argv):
    with pytest.raises(SystemExit) as e:
        cli.parse_args(argv)
    assert e.value.code == 2


def test_device_strategy_parses():
    spec = cli.parse_args(["bench", "--strategy", "device", "--devices", "4", "--gs-mode", "chaotic",
                           "--block-size", "8x8x8", "--roofline"])
    assert spec.strategy.kind == "device" and spec.strategy.devices == 4
    assert spec.strategy.resolved_gs_mode == "chaotic"
    assert spec.block_dims == (8, 8, 8) and spec.roofline
