"""The C-ABI library loads and exports every function include/psmooth.h
declares; the oracle's C restatement builds and agrees with the numpy one.
No device calls (CPU-only)."""

import ctypes
import os
import re

import numpy as np
import pytest

from oracle import restate as R

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _declared():
    text = open(os.path.join(ROOT, "include", "psmooth.h")).read()
    return sorted(set(re.findall(r"^(?:int|long long|const char\*)\s+(psm_\w+)\(", text, re.M)))


def test_header_declares_what_binding_uses():
    from paper_1208_1975_b200 import _lib

    assert _declared() == sorted(_lib.EXPORTS)


def test_library_exports_every_declared_symbol():
    from paper_1208_1975_b200 import _lib

    lib = _lib.load()
    for name in _declared():
        assert hasattr(lib, name), name
    assert lib.psm_version() >= 10000


def test_error_path_without_gpu_work():
    """Argument validation fails before any CUDA call and maps to ValueError."""
    from paper_1208_1975_b200 import _lib

    lib = _lib.load()
    out = ctypes.c_void_p()
    rc = lib.psm_plan_create(None, 0, None, 0, None, 0, None, ctypes.byref(out))
    assert rc == _lib.PSM_EINVAL
    with pytest.raises(ValueError):
        _lib.check(rc, "psm_plan_create")
    assert b"patch" in lib.psm_last_error()


def _c_oracle():
    path = os.path.join(ROOT, "oracle", "build", "liboracle.so")
    if not os.path.exists(path):
        pytest.skip("oracle C restatement not built (make -C oracle)")
    lib = ctypes.CDLL(path)
    lib.oracle_line_jacobi.restype = ctypes.c_double
    lib.oracle_line_jacobi.argtypes = [ctypes.c_void_p] * 3 + [ctypes.c_int] * 3 + [
        ctypes.c_double, ctypes.c_void_p, ctypes.c_double, ctypes.c_int, ctypes.c_int]
    return lib


@pytest.mark.parametrize("shape", [(48, 10, 9), (7, 3, 5), (256, 4, 3)])
def test_c_oracle_matches_numpy_oracle(shape):
    lib = _c_oracle()
    rng = np.random.default_rng(1)
    p = R.OPatch(shape)
    p.u[1:-1, 1:-1, 1:-1] = rng.standard_normal(shape)
    p.f[:] = rng.standard_normal(shape)
    lv = R.OLevel([p])
    lv.refresh_ghosts()
    u = np.asfortranarray(p.u.copy())
    f = np.asfortranarray(p.f.copy())
    v = np.zeros_like(u, order="F")
    faces = (ctypes.c_double * 6)(*R.DEFAULT_FACES)
    ss = lib.oracle_line_jacobi(u.ctypes.data, f.ctypes.data, v.ctypes.data, *shape, 6.0, faces, 0.8, 1, 2)
    r = R.residual(p.u, p.f)
    want = p.interior + 0.8 * R.line_solve(r)
    np.testing.assert_array_equal(v[1:-1, 1:-1, 1:-1], want)
    assert ss == pytest.approx(float(np.sum(r * r)), rel=1e-14)
