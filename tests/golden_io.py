"""Loading helpers for tests/golden/*.npz (made by oracle/make_golden.py from
the reference package itself)."""

import glob
import os

import numpy as np

GOLDEN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")


def load(name):
    with np.load(os.path.join(GOLDEN, name + ".npz"), allow_pickle=False) as d:
        return {k: d[k] for k in d.files}


def names(prefix=""):
    out = []
    for p in sorted(glob.glob(os.path.join(GOLDEN, prefix + "*.npz"))):
        out.append(os.path.splitext(os.path.basename(p))[0])
    return out


def single_patch_cases():
    return [n for n in names() if n.startswith(("line_", "plane_", "box_"))]


def multipatch_cases():
    return names("multi_")


def zsplit_cases():
    return names("zsplit_")


def rel_maxnorm(got, want):
    got = np.asarray(got)
    want = np.asarray(want)
    scale = max(float(np.max(np.abs(want))), 1e-300)
    return float(np.max(np.abs(got - want))) / scale


def hist_rel(got, want):
    return max(abs(a - b) / max(abs(b), 1e-300) for a, b in zip(got, want))
