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

__all__ = ["Stencil7", "FACE_OFFSETS", "assemble_block_matrix"]

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
