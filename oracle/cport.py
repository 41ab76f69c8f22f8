"""ctypes access to the C restatement (oracle/psm_oracle.c).

TEST INFRASTRUCTURE ONLY (see ``restate.py``'s header): used by ``tests/``
as a faster checker for full-size line-block configurations, where the numpy
restatement's Python-level wavefront loop would take minutes, and by
``bench.py``'s CPU legs.

``line_smooth`` follows ``restate.smooth`` (smoother.py:197-214): refresh
ghosts, history[0], then steps x (sweep, refresh, history entry).  The sweeps
are the C kernels: ``oracle_line_gs`` is the reference's serial lexicographic
block GS on one patch (smoother.py:156-169, runtime.py:164-168) and
``oracle_line_jacobi`` the snapshot Jacobi sweep (smoother.py:138-153).
Patches of one GS step are independent (their coupling is the step-end ghost
refresh), so they run on a thread pool; ctypes releases the GIL.
"""

from __future__ import annotations

import ctypes
import math
import os
from concurrent.futures import ThreadPoolExecutor

import numpy as np

from . import restate as R

_HERE = os.path.dirname(os.path.abspath(__file__))
_LIB = None


def load():
    global _LIB
    if _LIB is None:
        path = os.path.join(_HERE, "build", "liboracle.so")
        if not os.path.exists(path):
            raise RuntimeError(f"{path} missing: run `make -C oracle`")
        lib = ctypes.CDLL(path)
        dp, i, d = ctypes.c_void_p, ctypes.c_int, ctypes.c_double
        lib.oracle_line_gs.argtypes = [dp, dp, i, i, i, d, dp, d]
        lib.oracle_line_gs.restype = None
        lib.oracle_residual_sumsq.argtypes = [dp, dp, i, i, i, d, dp]
        lib.oracle_residual_sumsq.restype = d
        lib.oracle_line_jacobi.argtypes = [dp, dp, dp, i, i, i, d, dp, d, i, i]
        lib.oracle_line_jacobi.restype = d
        lib.oracle_fill_ghosts.argtypes = [dp, i, i, i, i]
        lib.oracle_fill_ghosts.restype = None
        lib.oracle_max_threads.restype = i
        _LIB = lib
    return _LIB


def _ptr(a):
    assert a.flags.f_contiguous and a.dtype == np.float64
    return ctypes.c_void_p(a.ctypes.data)


def _faces(faces):
    return (ctypes.c_double * 6)(*[float(c) for c in faces])


def residual_norm(level, center=R.DEFAULT_CENTER, faces=R.DEFAULT_FACES, pool=None):
    """sqrt of the per-patch sums of r^2, summed in patch order."""
    lib, fc = load(), _faces(faces)

    def one(p):
        nx, ny, nz = p.dims
        return lib.oracle_residual_sumsq(_ptr(p.u), _ptr(p.f), nx, ny, nz, float(center), fc)

    parts = list(pool.map(one, level.patches)) if pool is not None else [one(p) for p in level.patches]
    return math.sqrt(sum(parts))


def line_smooth(level, scheme, omega=None, steps=1, center=R.DEFAULT_CENTER, faces=R.DEFAULT_FACES,
                threads=None):
    """Line-block smooth of an ``R.OLevel`` in place; returns the history."""
    if omega is None:
        omega = 0.8 if scheme == "block_jacobi" else 1.0  # smoother.py:51
    lib, fc = load(), _faces(faces)
    threads = threads or os.cpu_count() or 1
    with ThreadPoolExecutor(threads) as pool:
        level.refresh_ghosts()
        hist = [residual_norm(level, center, faces, pool)]
        for _ in range(steps):
            if scheme == "block_jacobi":
                for p in level.patches:
                    nx, ny, nz = p.dims
                    lib.oracle_line_jacobi(_ptr(p.u), _ptr(p.f), _ptr(p.other), nx, ny, nz, float(center), fc,
                                           float(omega), 1, threads)
                for p in level.patches:
                    p.swap()
            else:
                def sweep(p):
                    nx, ny, nz = p.dims
                    lib.oracle_line_gs(_ptr(p.u), _ptr(p.f), nx, ny, nz, float(center), fc, float(omega))

                list(pool.map(sweep, level.patches))
            level.refresh_ghosts()
            hist.append(residual_norm(level, center, faces, pool))
    return hist
