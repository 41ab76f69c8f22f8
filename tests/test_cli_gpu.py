"""The device CLI (paper_1208_1975_b200.cli) against the reference CLI's own
CSV output on the same arguments (tests/golden/cli_*.csv, made by running
patchsmooth.cli): same header, same key columns, residual histories within
1e-12 relative; plus bench and inverses rows on the device."""

import csv
import io
import os

import pytest

from paper_1208_1975_b200 import cli

pytestmark = pytest.mark.gpu
GOLD = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")
CASES = sorted(f[:-4] for f in os.listdir(GOLD) if f.startswith("cli_") and f.endswith(".csv"))


def _run(argv, capsys):
    rc = cli.main(argv)
    out = capsys.readouterr().out
    assert rc == 0
    return out


@pytest.mark.parametrize("name", CASES)
def test_cli_matches_reference_csv(name, capsys):
    argv = open(os.path.join(GOLD, name + ".csv.args")).read().split()
    got = list(csv.reader(io.StringIO(_run(argv, capsys))))
    want = list(csv.reader(open(os.path.join(GOLD, name + ".csv"))))
    assert got[0] == want[0] and len(got) == len(want)
    for g, w in zip(got[1:], want[1:]):
        assert g[:5] == w[:5]  # scheme, block, patch, seed, step
        for a, b in zip(g[5:], w[5:]):
            assert abs(float(a) - float(b)) <= 1e-12 * abs(float(b)), (name, g, w)


def test_cli_bench_rows(capsys):
    out = _run(["bench", "--patch-size", "32x16x16", "--block-size", "32x1x1", "--strategy", "device",
                "--steps", "2", "--repeat", "2", "--roofline"], capsys)
    rows = list(csv.reader(io.StringIO(out)))
    assert rows[0][-1] == "gbytes_per_second"
    assert [r[3] for r in rows[1:]] == ["serial", "device"]
    assert float(rows[1][10]) == 1.0 and float(rows[1][11]) == 1.0
    assert all(float(r[8]) > 0 and float(r[12]) > 0 for r in rows[1:])


def test_cli_inverses_multiply_back(capsys):
    out = _run(["inverses", "--patch-size", "12x10x8", "--block-size", "8x8x8"], capsys)
    rows = list(csv.reader(io.StringIO(out)))
    assert rows[0] == ["block", "extent", "order", "invert_seconds", "multiply_back_inf_error"]
    assert {r[1] for r in rows[1:]} == {"8x8x8", "4x8x8", "8x2x8", "4x2x8"}
    assert all(float(r[4]) < 1e-12 for r in rows[1:])


def test_cli_argument_errors_exit_2():
    with pytest.raises(SystemExit) as e:
        cli.main(["smooth", "--devices", "2"])
    assert e.value.code == 2
