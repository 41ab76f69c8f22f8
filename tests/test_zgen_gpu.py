"""Line Jacobi through the z-marching kernel with a runtime line length
(psm_line_zgen.cu, any even nx in [42, 1024]) against the CPU restatement:
iterates within 1e-12 relative max-norm, ghosts included, and the history.

The kernel is chosen for plane groups of at least PSM_ZMARCH_MIN_CELLS cells
(default 2^21); the small cases run in a child process with the threshold at
0, the large one (a 130^3 patch) in this process at the default."""

import os

import numpy as np
import pytest
import torch
import torch.multiprocessing as mp

import golden_io as G
from oracle import restate as R

pytestmark = pytest.mark.gpu
TOL = 1e-12
STEPS = 3
# single patches and a mixed-nx level (patches abutting along x, partial faces)
SMALL = [
    [((72, 40, 30), (0, 0, 0))],
    [((96, 33, 20), (0, 0, 0))],
    [((250, 9, 7), (0, 0, 0))],
    [((1000, 3, 4), (0, 0, 0))],
    [((42, 50, 6), (0, 0, 0))],
    [((88, 21, 11), (0, 0, 0)), ((80, 24, 11), (88, 0, 0)), ((72, 16, 9), (168, 3, 1))],
]


def _inputs(specs, seed):
    rng = np.random.default_rng(seed)
    return [rng.standard_normal(d) for d, _ in specs], [rng.standard_normal(d) for d, _ in specs]


def _device_run(specs, seed, omega, stencil=None):
    import paper_1208_1975_b200 as ps

    u0, f = _inputs(specs, seed)
    patches = [ps.Patch(ps.PatchDims(*d), o) for d, o in specs]
    for p, a, b in zip(patches, u0, f):
        p.interior[...] = torch.from_numpy(a).cuda()
        p.f[...] = torch.from_numpy(b).cuda()
    kw = {} if stencil is None else {"stencil": ps.Stencil7(*stencil)}
    nxmax = max(d[0] for d, _ in specs)
    cfg = ps.SmootherConfig(scheme="block_jacobi", block_dims=(nxmax, 1, 1), omega=omega, steps=STEPS, **kw)
    _, hist = ps.smooth(ps.Level(patches), cfg, ps.InverseCache())
    return [p.u.cpu().numpy() for p in patches], hist


def _oracle_run(specs, seed, omega, stencil=None):
    u0, f = _inputs(specs, seed)
    ops = []
    for (d, o), a, b in zip(specs, u0, f):
        op = R.OPatch(d, o)
        op.u[1:-1, 1:-1, 1:-1] = a
        op.f[:] = b
        ops.append(op)
    nxmax = max(d[0] for d, _ in specs)
    kw = {} if stencil is None else {"center": stencil[0], "faces": stencil[1]}
    hist = R.smooth(R.OLevel(ops), "block_jacobi", (nxmax, 1, 1), omega=omega, steps=STEPS, **kw)
    return [op.u for op in ops], hist


CASES = [(i, 0.8, None) for i in range(len(SMALL))] + [(0, 0.6, (7.0, (-1.2, -0.9, -1.0, -1.0, -1.1, -0.8)))]


def _child(rank, out_dir):
    os.environ["PSM_ZMARCH_MIN_CELLS"] = "0"
    torch.cuda.set_device(0)
    for c, (i, omega, stencil) in enumerate(CASES):
        us, hist = _device_run(SMALL[i], 100 + i, omega, stencil)
        np.savez(os.path.join(out_dir, f"zgen{c}.npz"), hist=np.array(hist), *us)


def test_zgen_small_shapes_match_oracle(tmp_path):
    mp.spawn(_child, args=(str(tmp_path),), nprocs=1, join=True)
    for c, (i, omega, stencil) in enumerate(CASES):
        with np.load(tmp_path / f"zgen{c}.npz") as d:
            got = [d[f"arr_{k}"] for k in range(len(SMALL[i]))]
            hist = d["hist"]
        want, want_hist = _oracle_run(SMALL[i], 100 + i, omega, stencil)
        for g, w in zip(got, want):
            assert G.rel_maxnorm(g[1:-1, 1:-1, 1:-1], w[1:-1, 1:-1, 1:-1]) < TOL, (c, SMALL[i])
            assert G.rel_maxnorm(g, w) < TOL, (c, "ghosts")
        assert G.hist_rel(hist, want_hist) < TOL


def test_zgen_default_threshold_130_cubed():
    specs = [((130, 130, 130), (0, 0, 0))]
    got, hist = _device_run(specs, 7, 0.8)
    want, want_hist = _oracle_run(specs, 7, 0.8)
    assert G.rel_maxnorm(got[0], want[0]) < TOL
    assert G.hist_rel(hist, want_hist) < TOL
