"""ctypes binding of libpsmooth.so (the C ABI declared in include/psmooth.h).

The library is built in-tree (``make`` or ``__graft_entry__.build()``) and
loaded from this package directory.  There is no fallback: if the library or
a CUDA device is missing, every smoothing call raises.
"""

from __future__ import annotations

import ctypes
import os
import threading

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("PSM_LIB", os.path.join(_HERE, "libpsmooth.so"))  # override: tools/profiling builds

PSM_OK = 0
PSM_EINVAL = -1
PSM_ESINGULAR = -2
PSM_ECUDA = -3
PSM_ENOMEM = -4
PSM_EUNSUPPORTED = -5

BLOCK_LINE = 1
BLOCK_PLANE = 2
BLOCK_BOX = 3
GHOST_PHYSICAL = 1
GHOST_INTERFACE = 2
GHOST_SKIP_X = 4
GHOST_ALL = 3
GS_WAVEFRONT = 0
GS_CHAOTIC = 1

# every symbol include/psmooth.h declares (checked by tests/test_lib_exports.py)
EXPORTS = (
    "psm_last_error",
    "psm_version",
    "psm_factors_create",
    "psm_factors_create_box",
    "psm_factors_destroy",
    "psm_factors_apply",
    "psm_plan_create",
    "psm_plan_destroy",
    "psm_plan_reserve_history",
    "psm_refresh_ghosts",
    "psm_residual",
    "psm_jacobi_sweep",
    "psm_gs_sweep",
    "psm_history_sumsq",
    "psm_history_planes",
    "psm_tree_sum",
    "psm_jacobi_sweep_planes",
    "psm_halo_unpack",
    "psm_plan_launches",
    "psm_plane_solver",
    "psm_smooth_steps",
    "psm_device_pci_bus_id",
    "psm_peer_access",
    "psm_ipc_get_handle",
    "psm_ipc_open_handle",
    "psm_ipc_close_all",
    "psm_plan_set_peer_halo",
    "psm_halo_signal",
    "psm_halo_wait",
    "psm_box_residual",
    "psm_matvec",
    "psm_invert_dense",
)
PLANE_AUTO = 0
PLANE_DST = 1


class Stencil(ctypes.Structure):
    _fields_ = [("center", ctypes.c_double), ("faces", ctypes.c_double * 6)]


class PatchDesc(ctypes.Structure):
    _fields_ = [
        ("buf", ctypes.c_void_p * 2),
        ("f", ctypes.c_void_p),
        ("nx", ctypes.c_int),
        ("ny", ctypes.c_int),
        ("nz", ctypes.c_int),
    ]


class CopyDesc(ctypes.Structure):
    _fields_ = [
        ("src", ctypes.c_int),
        ("dst", ctypes.c_int),
        ("src_lo", ctypes.c_int * 3),
        ("dst_lo", ctypes.c_int * 3),
        ("extent", ctypes.c_int * 3),
    ]


class LibraryError(RuntimeError):
    """A CUDA or library failure inside libpsmooth."""


_lib = None
_lock = threading.Lock()


def load():
    """Load libpsmooth.so once; raise loudly when it is missing."""
    global _lib
    if _lib is not None:
        return _lib
    with _lock:
        if _lib is not None:
            return _lib
        if not os.path.exists(LIB_PATH):
            raise LibraryError(
                f"{LIB_PATH} not built; run `make` (or __graft_entry__.build()) -- "
                "there is no CPU fallback"
            )
        lib = ctypes.CDLL(LIB_PATH)
        vp, i, d, ll = ctypes.c_void_p, ctypes.c_int, ctypes.c_double, ctypes.c_longlong
        ub = ctypes.POINTER(ctypes.c_ubyte)
        sig = {
            "psm_last_error": (ctypes.c_char_p, []),
            "psm_version": (i, []),
            "psm_factors_create": (i, [i, ctypes.POINTER(Stencil), i, i, ctypes.POINTER(vp)]),
            "psm_factors_create_box": (i, [ctypes.POINTER(Stencil), i, i, i, ctypes.POINTER(vp)]),
            "psm_factors_destroy": (i, [vp]),
            "psm_factors_apply": (i, [vp, vp, vp, ll, vp]),
            "psm_plan_create": (
                i,
                [ctypes.POINTER(PatchDesc), i, ctypes.POINTER(CopyDesc), i, ctypes.POINTER(Stencil), i,
                 ctypes.POINTER(vp), ctypes.POINTER(vp)],
            ),
            "psm_plan_destroy": (i, [vp]),
            "psm_plan_reserve_history": (i, [vp, i]),
            "psm_refresh_ghosts": (i, [vp, ub, i, vp]),
            "psm_residual": (i, [vp, ub, i, vp]),
            "psm_jacobi_sweep": (i, [vp, ub, d, i, vp]),
            "psm_gs_sweep": (i, [vp, ub, d, i, vp]),
            "psm_history_sumsq": (i, [vp, i, ctypes.POINTER(d), vp]),
            "psm_history_planes": (i, [vp, i, vp, vp]),
            "psm_tree_sum": (i, [vp, ll, vp, vp]),
            "psm_jacobi_sweep_planes": (i, [vp, ub, d, i, i, i, i, vp]),
            "psm_halo_unpack": (i, [vp, ub, i, i, vp, vp]),
            "psm_plan_launches": (ll, [vp]),
            "psm_plane_solver": (i, [i]),
            "psm_smooth_steps": (i, [vp, ub, i, d, i, i, i, vp]),
            "psm_device_pci_bus_id": (i, [ctypes.c_char_p, i]),
            "psm_peer_access": (i, [ctypes.c_char_p, ctypes.POINTER(i)]),
            "psm_ipc_get_handle": (i, [vp, vp, ctypes.POINTER(ll)]),
            "psm_ipc_open_handle": (i, [vp, ll, ctypes.POINTER(vp)]),
            "psm_ipc_close_all": (i, []),
            "psm_plan_set_peer_halo": (i, [vp, i, i, vp, vp, i]),
            "psm_halo_signal": (i, [vp, vp, i, vp]),
            "psm_halo_wait": (i, [vp, i, i, vp]),
            "psm_box_residual": (i, [vp, vp, i, i, i, ctypes.POINTER(i), ctypes.POINTER(i), ctypes.POINTER(Stencil),
                                     vp, vp]),
            "psm_matvec": (i, [vp, vp, vp, d, vp, i, vp]),
            "psm_invert_dense": (i, [vp, i, vp, ctypes.POINTER(i), ctypes.POINTER(d), vp]),
        }
        for name, (res, args) in sig.items():
            if "PSM_LIB" in os.environ and not hasattr(lib, name):
                continue  # an older / profiling build named explicitly: bind what it has
            fn = getattr(lib, name)
            fn.restype = res
            fn.argtypes = args
        _lib = lib
        return lib


def check(rc, what=""):
    """Map a psm_status to the reference's exception types."""
    if rc == PSM_OK:
        return
    msg = load().psm_last_error().decode(errors="replace")
    text = f"{what}: {msg}" if what else msg
    if rc == PSM_EINVAL:
        raise ValueError(text)
    if rc == PSM_ESINGULAR:
        from .blocklinalg import SingularMatrixError

        raise SingularMatrixError(text)
    if rc == PSM_EUNSUPPORTED:
        raise ValueError(text)
    raise LibraryError(f"{text} (status {rc})")


def active_array(flags):
    arr = (ctypes.c_ubyte * len(flags))(*flags)
    return arr
