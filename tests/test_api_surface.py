"""The public surface is a superset of the reference's (drop-in imports):
every name in patchsmooth.__all__ exists here, and every public callable
takes the reference's positional parameters first, in the same order.
Pinned to tests/golden/api_surface.json (oracle/make_api_golden.py ran the
reference's own package); also checked live when the reference is present."""

import inspect
import json
import os
import sys

import pytest

import paper_1208_1975_b200 as ps

GOLD = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden", "api_surface.json")
REF = "/root/reference/pkg/src"


def _surface():
    with open(GOLD) as fh:
        return json.load(fh)


def test_reference_names_importable():
    ref = _surface()
    missing = sorted(set(ref["all"]) - set(ps.__all__))
    assert not missing, missing
    for name in ref["all"]:
        assert hasattr(ps, name), name


@pytest.mark.parametrize("name", sorted(_surface()["signatures"]))
def test_reference_signature_prefix(name):
    want = _surface()["signatures"][name]
    got = list(inspect.signature(getattr(ps, name)).parameters)
    assert got[: len(want)] == want, (name, got, want)


@pytest.mark.skipif(not os.path.isdir(REF), reason="reference not present")
def test_fixture_matches_live_reference():
    sys.path.insert(0, REF)
    try:
        import patchsmooth
    finally:
        sys.path.remove(REF)
    assert sorted(patchsmooth.__all__) == sorted(_surface()["all"])
