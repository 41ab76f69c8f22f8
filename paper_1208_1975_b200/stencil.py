"""The constant-coefficient 7-point stencil (reference ``stencil.py:52-68``).

Only the coefficient record lives here; the operator itself is applied inside
the sm_100a kernels, in the reference's operation order (``stencil.py:106-111``:
``acc = c*u``, then ``acc += face*neighbour`` for -x,+x,-y,+y,-z,+z, then
``r = f - acc``), so device residuals are bit-identical to the reference's
for the same field values.
"""

from __future__ import annotations

import math
from dataclasses import dataclass

from . import _lib

__all__ = ["Stencil7", "FACE_OFFSETS", "assemble_block_matrix", "assemble_patch_matrix", "apply_stencil",
           "block_residual"]

_MAX_DENSE = 32768  # stencil.py:39

# stencil.py:42-49
FACE_OFFSETS = ((-1, 0, 0), (1, 0, 0), (0, -1, 0), (0, 1, 0), (0, 0, -1), (0, 0, 1))


@dataclass(frozen=True)
class Stencil7:
    """Center coefficient plus six face coefficients (-x,+x,-y,+y,-z,+z)."""

    center: float = 6.0
    faces: tuple = (-1.0, -1.0, -1.0, -1.0, -1.0, -1.0)

    def __post_init__(self):
        object.__setattr__(self, "center", float(self.center))
        faces = tuple(float(c) for c in self.faces)
        object.__setattr__(self, "faces", faces)
        if len(faces) != 6:
            raise ValueError(f"need exactly 6 face coefficients, got {len(faces)}")
        if not all(math.isfinite(c) for c in (self.center, *faces)):
            raise ValueError("stencil coefficients must be finite")
        if not self.center > 0:
            raise ValueError(f"center coefficient must be positive, got {self.center}")

    def _cstruct(self):
        s = _lib.Stencil()
        s.center = self.center
        for i, c in enumerate(self.faces):
            s.faces[i] = c
        return s


def assemble_block_matrix(stencil, extent, device=None):
    """Dense operator of one block, couplings inside the block only
    (stencil.py:115-138), cells x fastest, as a float64 tensor on ``device``
    (for the ``inverses`` report and multiply-back checks; the smoother never
    forms it)."""
    import torch

    from .grid import _int3, default_device

    ex, ey, ez = _int3(extent, "extent")
    if min(ex, ey, ez) < 1:
        raise ValueError(f"extent must be positive, got {(ex, ey, ez)}")
    dev = torch.device(device) if device is not None else default_device()
    n = ex * ey * ez
    a = torch.zeros((n, n), dtype=torch.float64, device=dev)
    idx = torch.arange(n, device=dev)
    x, y, z = idx % ex, (idx // ex) % ey, idx // (ex * ey)
    a[idx, idx] = stencil.center
    for c, (dx, dy, dz) in zip(stencil.faces, FACE_OFFSETS):
        px, py, pz = x + dx, y + dy, z + dz
        ok = (px >= 0) & (px < ex) & (py >= 0) & (py < ey) & (pz >= 0) & (pz < ez)
        a[idx[ok], (px + ex * (py + ey * pz))[ok]] = c
    return a


def _box_on_device(stencil, patch, lo, ext, with_f):
    """f - A u (with_f) or A u on the interior box [lo, lo+ext) of ``patch``'s
    active buffer, flattened x fastest, by psm_box_residual."""
    import ctypes

    import torch

    if patch.dims.ghost_width != 1:
        raise ValueError("stencil application requires ghost_width == 1")
    dev = patch.device
    if dev.type != "cuda":
        raise RuntimeError("stencil application runs on the CUDA device (no CPU fallback)")
    n = ext[0] * ext[1] * ext[2]
    out = torch.empty(n, dtype=torch.float64, device=dev)
    lo_c, ext_c = (ctypes.c_int * 3)(*lo), (ctypes.c_int * 3)(*ext)
    st = stencil._cstruct()
    with torch.cuda.device(dev):
        stream = ctypes.c_void_p(torch.cuda.current_stream(dev).cuda_stream)
        _lib.check(_lib.load().psm_box_residual(
            ctypes.c_void_p(patch._bufs[patch._active].data_ptr()),
            ctypes.c_void_p(patch._f.data_ptr()) if with_f else None,
            *patch.dims.shape, lo_c, ext_c, ctypes.byref(st), ctypes.c_void_p(out.data_ptr()), stream),
            "box_residual")
    return out


def apply_stencil(stencil, patch, coords):
    """Pointwise A u at one interior cell, ghosts read as stored
    (stencil.py:71-84); computed on the patch's device."""
    from .grid import _int3

    if patch.dims.ghost_width != 1:
        raise ValueError("stencil application requires ghost_width == 1")
    i, j, k = _int3(coords, "coords")
    nx, ny, nz = patch.dims.shape
    if not (0 <= i < nx and 0 <= j < ny and 0 <= k < nz):
        raise ValueError(f"coords {coords!r} outside the interior box")
    return float(_box_on_device(stencil, patch, (i, j, k), (1, 1, 1), False)[0])


def block_residual(stencil, patch, block):
    """f - A u restricted to ``block`` (a BlockRange), flattened x fastest,
    ghosts read as stored (stencil.py:93-112).  Returns a float64 tensor on
    the patch's device, bit-identical to the reference's numpy result."""
    from .grid import BlockRange

    if patch.dims.ghost_width != 1:
        raise ValueError("block residual requires ghost_width == 1")
    if not isinstance(block, BlockRange):
        raise TypeError(f"block must be a BlockRange, got {type(block).__name__}")
    if any(h > n for h, n in zip(block.hi, patch.dims.shape)):
        raise ValueError(f"block {block} leaves the interior {patch.dims.shape}")
    return _box_on_device(stencil, patch, block.lo, block.extent, True)


def assemble_patch_matrix(stencil, dims, device=None):
    """Dense interior operator of one patch with every face physical
    (stencil.py:141-168): the ghost rule ghost = -interior folds each coupling
    that leaves the patch into the diagonal (center - sum of those faces).
    Cells x fastest; built on ``device``; capped at 32768 cells."""
    import torch

    from .grid import PatchDims, default_device

    if not isinstance(dims, PatchDims):
        raise TypeError(f"dims must be a PatchDims, got {type(dims).__name__}")
    m = dims.interior_cells
    if m > _MAX_DENSE:
        raise ValueError(f"patch has {m} cells, dense assembly capped at {_MAX_DENSE}")
    nx, ny, nz = dims.shape
    dev = torch.device(device) if device is not None else default_device()
    idx = torch.arange(m, device=dev)
    x, y, z = idx % nx, (idx // nx) % ny, idx // (nx * ny)
    a = torch.zeros((m, m), dtype=torch.float64, device=dev)
    diag = torch.full((m,), stencil.center, dtype=torch.float64, device=dev)
    for c, (dx, dy, dz) in zip(stencil.faces, FACE_OFFSETS):
        px, py, pz = x + dx, y + dy, z + dz
        inside = (px >= 0) & (px < nx) & (py >= 0) & (py < ny) & (pz >= 0) & (pz < nz)
        a[idx[inside], (px + nx * (py + ny * pz))[inside]] = c
        diag = torch.where(inside, diag, diag - c)
    a[idx, idx] = diag
    return a
