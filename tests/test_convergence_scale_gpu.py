"""SURVEY f4 at scale: thousands of damped block-Jacobi sweeps on patches
the reference's dense spectral oracle cannot handle (48^3 and 64^3 line
blocks, 32^3 plane blocks), against the exact spectral radius of the
iteration, computed here by separation of variables.

The smoother's error propagator is G = I - omega M^-1 A, where A is the
7-point operator with the odd-reflection ghosts (ghost = -interior,
grid.py:311-330: +1 on the diagonal of every boundary cell per face) and M
the closure-free block (stencil.py:115-138: no reflections; they stay in the
lagged residual).  The directions outside the block are diagonal in the
DST-II basis of the reflected 1-D operator (eigenvalues 2 - 2 cos(pi m / n)),
so rho(G) is the largest spectral radius of small dense problems, one per
outer mode.  The same reduction reproduces the reference's dense
power-iteration values (test_analysis.py: 8^3 line 0.911618881, 12^3 line
0.959740910, 8^3 plane 0.839037027) to 1e-7, checked in the first test."""

import math

import numpy as np
import pytest

import paper_1208_1975_b200 as ps

pytestmark = pytest.mark.gpu


def _tri(n, off, diag):
    return np.diag(np.full(n, float(diag))) + np.diag(np.full(n - 1, float(off)), 1) + np.diag(
        np.full(n - 1, float(off)), -1)


def _refl(n):
    r = np.zeros((n, n))
    r[0, 0] = r[-1, -1] = 1.0
    return r


def rho_line(n, omega=0.8):
    best = 0.0
    for j, k in ((1, 1), (1, 2), (2, 2)):
        shift = 6 - 2 * math.cos(math.pi * j / n) - 2 * math.cos(math.pi * k / n)
        a = shift * np.eye(n) + _tri(n, -1, 0) + _refl(n)
        g = np.eye(n) - omega * np.linalg.solve(_tri(n, -1, 6), a)
        best = max(best, float(np.max(np.abs(np.linalg.eigvals(g)))))
    return best


def rho_plane(n, omega=0.8):
    eye, s, r = np.eye(n), _tri(n, 1, 0), _refl(n)
    m = 6 * np.eye(n * n) - np.kron(s, eye) - np.kron(eye, s)
    best = 0.0
    for k in (1, 2):
        a = m - 2 * math.cos(math.pi * k / n) * np.eye(n * n) + np.kron(r, eye) + np.kron(eye, r)
        g = np.eye(n * n) - omega * np.linalg.solve(m, a)
        best = max(best, float(np.max(np.abs(np.linalg.eigvals(g)))))
    return best


def test_reduction_reproduces_reference_oracle_values():
    assert rho_line(8) == pytest.approx(0.911618881, abs=2e-7)
    assert rho_line(12) == pytest.approx(0.959740910, abs=2e-7)
    assert rho_plane(8) == pytest.approx(0.839037027, abs=2e-7)


@pytest.mark.parametrize("n,block,steps", [(48, "line", 3000), (64, "line", 5000), (32, "plane", 1500)])
def test_jacobi_asymptotic_factor_at_scale(n, block, steps):
    rho = rho_line(n) if block == "line" else rho_plane(n)
    bd = (n, 1, 1) if block == "line" else (n, n, 1)
    rep, = ps.run_convergence_study(ps.PatchDims(n, n, n), block_sizes=[bd], schemes=["block_jacobi"], steps=steps,
                                    window=(steps // 2, steps // 2 - 1))
    assert rep.residual_history[-1] / rep.residual_history[0] > 1e-12  # window above the rounding floor
    assert rep.asymptotic_factor == pytest.approx(rho, rel=5e-4), (rep.asymptotic_factor, rho)
