"""Synthetic levels and inputs (reference ``bench.py:106-146``).

``build_level`` and ``seed_initial_guess`` keep the reference's layout and
random stream exactly (patches along x; u0 ~ U[0,1) from one
``default_rng(seed)`` in patch order, drawn as a C-order (nx,ny,nz) array;
f = 0), so the same seed gives the same starting field as the reference.
``build_lattice`` is the AMR-style a x b x c lattice of equal patches used
for the multi-patch configuration.
"""

from __future__ import annotations

import itertools
import os

import numpy as np
import torch

from .grid import Level, Patch, PatchDims, _int3

__all__ = ["build_level", "build_lattice", "seed_initial_guess", "cells_smoothed", "allocation_cap"]


CAP_ENV = "PATCHSMOOTH_MAX_CELLS"  # bench.py:40-41
DEFAULT_CAP = 300_000_000


def allocation_cap():
    """Cell cap for build_level: $PATCHSMOOTH_MAX_CELLS or 3e8 (bench.py:93-103).
    The device holds far more (180 GB); raise the variable for big levels."""
    raw = os.environ.get(CAP_ENV)
    if raw is None:
        return DEFAULT_CAP
    try:
        cap = int(raw)
    except ValueError:
        raise ValueError(f"{CAP_ENV} must be an integer, got {raw!r}") from None
    if cap < 1:
        raise ValueError(f"{CAP_ENV} must be positive, got {cap}")
    return cap


def build_level(sizes, max_cells=None, device=None):
    """Patches of the given interior sizes abutting end to end along x
    (bench.py:106-131).  Allocation (two padded buffers plus f per patch)
    must fit ``max_cells`` (default: ``allocation_cap()``)."""
    dims = [PatchDims(*_int3(s, "patch size")) for s in sizes]
    if not dims:
        raise ValueError("no patch sizes given")
    cap = allocation_cap() if max_cells is None else max_cells
    need = sum(2 * d.total_cells + d.interior_cells for d in dims)
    if need > cap:
        raise ValueError(f"patch set needs {need} cells, cap is {cap} (raise {CAP_ENV} to allow it)")
    origins = itertools.accumulate([0] + [d.nx for d in dims[:-1]])
    return Level([Patch(d, origin=(x0, 0, 0), device=device) for d, x0 in zip(dims, origins)])


def build_lattice(counts, size, device=None):
    """counts[0] x counts[1] x counts[2] equal patches, x fastest in patch order."""
    a, b, c = _int3(counts, "counts")
    size = _int3(size, "size")
    patches = [
        Patch(PatchDims(*size), origin=(i * size[0], j * size[1], k * size[2]), device=device)
        for k in range(c)
        for j in range(b)
        for i in range(a)
    ]
    return Level(patches)


def seed_initial_guess(level, seed):
    """Interior ~ U[0,1) from one generator in patch order; f untouched
    (bench.py:141-146)."""
    rng = np.random.default_rng(seed)
    for p in level.patches:
        vals = rng.random(p.dims.shape)
        p.interior[...] = torch.from_numpy(vals).to(p.device)
    return level


def cells_smoothed(level, steps):
    if not isinstance(steps, int) or isinstance(steps, bool) or steps < 1:
        raise ValueError(f"steps must be a positive integer, got {steps!r}")
    return steps * level.interior_cells
