"""Patches, levels and ghost layers on the device.

Mirrors ``patchsmooth.grid`` (reference ``grid.py:1-547``): the same class
and function names, the same index conventions and the same memory order, but
every field is a CUDA ``torch.float64`` tensor and ghost work runs in
``libpsmooth`` kernels.

Memory layout.  The reference stores u as a numpy Fortran-ordered
``(nx+2, ny+2, nz+2)`` array (x fastest, ``grid.py:177-182``).  Here each
buffer is a C-contiguous ``(nz+2, ny+2, nx+2)`` tensor -- byte-for-byte the
same order -- and ``Patch.u`` returns it permuted to ``[i, j, k]`` indexing,
so ``p.u[1:-1, 1:-1, 1:-1] = ...`` reads exactly like reference code.  f is
``(nz, ny, nx)`` exposed as ``[i, j, k]``; its storage never moves (assigning
``p.f = a`` copies into it) because device plans hold raw pointers.
"""

from __future__ import annotations

import ctypes
import itertools
from dataclasses import dataclass

import numpy as np
import torch

from . import _lib

__all__ = [
    "PatchDims",
    "Patch",
    "BlockRange",
    "BlockDecomposition",
    "InterfaceCopy",
    "Level",
    "global_index",
    "block_cell",
    "ghost_overhead",
    "decompose_blocks",
    "fill_physical_ghosts",
    "exchange_interface_ghosts",
    "default_device",
]

_MAX_LINEAR = 2**62  # grid.py:50-51


def default_device():
    """The device new patches live on: the current CUDA device, else CPU
    (CPU patches support construction and host-side logic only)."""
    if torch.cuda.is_available():
        return torch.device("cuda", torch.cuda.current_device())
    return torch.device("cpu")


def _int3(value, name):
    try:
        triple = tuple(int(c) for c in value)
    except TypeError:
        raise ValueError(f"{name} must be a triple of integers, got {value!r}") from None
    if len(triple) != 3:
        raise ValueError(f"{name} must have exactly 3 entries, got {value!r}")
    return triple


@dataclass(frozen=True)
class PatchDims:
    """Interior extents plus ghost width (grid.py:64-111)."""

    nx: int
    ny: int
    nz: int
    ghost_width: int = 1

    def __post_init__(self):
        for name in ("nx", "ny", "nz"):
            n = getattr(self, name)
            if isinstance(n, bool) or not isinstance(n, (int, np.integer)) or n < 1:
                raise ValueError(f"{name} must be a positive integer, got {n!r}")
        if self.ghost_width not in (0, 1):
            raise ValueError(f"ghost_width must be 0 or 1, got {self.ghost_width!r}")
        if self.total_cells > _MAX_LINEAR:
            raise ValueError("padded patch exceeds the linear index space")

    @property
    def shape(self):
        return (self.nx, self.ny, self.nz)

    @property
    def padded_shape(self):
        w = 2 * self.ghost_width
        return (self.nx + w, self.ny + w, self.nz + w)

    @property
    def interior_cells(self):
        return self.nx * self.ny * self.nz

    @property
    def total_cells(self):
        a, b, c = self.padded_shape
        return a * b * c


def global_index(dims, coords, with_ghost=False):
    """Linear x-fastest offset of a cell (grid.py:114-130)."""
    i, j, k = _int3(coords, "coords")
    g = dims.ghost_width
    if with_ghost:
        px, py, pz = dims.padded_shape
        if not all(-g <= c < n + g for c, n in zip((i, j, k), dims.shape)):
            raise ValueError(f"coords {coords!r} outside the padded box")
        return (i + g) + px * ((j + g) + py * (k + g))
    if not all(0 <= c < n for c, n in zip((i, j, k), dims.shape)):
        raise ValueError(f"coords {coords!r} outside the interior box")
    return i + dims.nx * (j + dims.ny * k)


def block_cell(block_index, block_dims, local):
    """Interior coordinates of an in-block cell (grid.py:133-143)."""
    b = _int3(block_index, "block_index")
    d = _int3(block_dims, "block_dims")
    t = _int3(local, "local")
    return tuple(bi * di + ti for bi, di, ti in zip(b, d, t))


def ghost_overhead(dims):
    """(ghost cells, ghost/interior) (grid.py:146-150)."""
    ghosts = dims.total_cells - dims.interior_cells
    return ghosts, ghosts / dims.interior_cells


class Patch:
    """Two padded device buffers (active u, staging v) plus interior f.

    Same contract as the reference Patch (grid.py:153-217): ``u`` is the
    active padded field, ``v`` the interior of the inactive one,
    ``swap_buffers`` flips roles without copying.
    """

    __slots__ = ("dims", "origin", "_bufs", "_active", "_f", "__weakref__")

    def __init__(self, dims, origin=(0, 0, 0), device=None):
        if not isinstance(dims, PatchDims):
            raise TypeError(f"dims must be a PatchDims, got {type(dims).__name__}")
        self.dims = dims
        self.origin = _int3(origin, "origin")
        dev = torch.device(device) if device is not None else default_device()
        px, py, pz = dims.padded_shape
        self._bufs = (
            torch.zeros((pz, py, px), dtype=torch.float64, device=dev),
            torch.zeros((pz, py, px), dtype=torch.float64, device=dev),
        )
        self._active = 0
        self._f = torch.zeros((dims.nz, dims.ny, dims.nx), dtype=torch.float64, device=dev)

    @property
    def device(self):
        return self._f.device

    @property
    def u(self):
        """Active padded field, indexed [i, j, k] with ghost offset +1."""
        return self._bufs[self._active].permute(2, 1, 0)

    @property
    def v(self):
        """Interior view of the inactive (staging) buffer."""
        return self._bufs[1 - self._active].permute(2, 1, 0)[self._interior_slices]

    @property
    def interior(self):
        return self.u[self._interior_slices]

    @property
    def f(self):
        """Right-hand side, interior only, indexed [i, j, k]."""
        return self._f.permute(2, 1, 0)

    @f.setter
    def f(self, value):
        self.f[...] = torch.as_tensor(np.asarray(value) if not torch.is_tensor(value) else value,
                                      dtype=torch.float64).to(self._f.device)

    @property
    def _interior_slices(self):
        g = self.dims.ghost_width
        return tuple(slice(g, g + n) for n in self.dims.shape)

    def swap_buffers(self):
        self._active = 1 - self._active

    @property
    def global_box(self):
        return tuple((o, o + n) for o, n in zip(self.origin, self.dims.shape))

    def _desc(self):
        d = _lib.PatchDesc()
        d.buf[0] = self._bufs[0].data_ptr()
        d.buf[1] = self._bufs[1].data_ptr()
        d.f = self._f.data_ptr()
        d.nx, d.ny, d.nz = self.dims.shape
        return d

    def __repr__(self):
        nx, ny, nz = self.dims.shape
        return f"Patch({nx}x{ny}x{nz} at {self.origin})"


@dataclass(frozen=True)
class BlockRange:
    """Half-open cell range (grid.py:220-251)."""

    lo: tuple
    extent: tuple

    def __post_init__(self):
        object.__setattr__(self, "lo", _int3(self.lo, "lo"))
        object.__setattr__(self, "extent", _int3(self.extent, "extent"))
        if min(self.lo) < 0:
            raise ValueError(f"block lo must be non-negative, got {self.lo}")
        if min(self.extent) < 1:
            raise ValueError(f"block extent must be positive, got {self.extent}")

    @property
    def hi(self):
        return tuple(a + b for a, b in zip(self.lo, self.extent))

    @property
    def cells(self):
        return int(np.prod(self.extent))

    def slices(self, offset=0):
        return tuple(slice(a + offset, a + b + offset) for a, b in zip(self.lo, self.extent))


@dataclass(frozen=True)
class BlockDecomposition:
    """Blocks of one patch, lexicographic x fastest (grid.py:254-283)."""

    block_dims: tuple
    counts: tuple
    ranges: tuple

    @property
    def shapes(self):
        return tuple(dict.fromkeys(r.extent for r in self.ranges))

    def block_of(self, coords):
        c = _int3(coords, "coords")
        idx = [ci // bi for ci, bi in zip(c, self.block_dims)]
        if not all(0 <= a < n for a, n in zip(idx, self.counts)):
            raise ValueError(f"coords {coords!r} outside the decomposed interior")
        return idx[0] + self.counts[0] * (idx[1] + self.counts[1] * idx[2])


def decompose_blocks(dims, block_dims):
    """ceil(n/b) ranges per axis, trailing ranges truncated (grid.py:286-308)."""
    if not isinstance(dims, PatchDims):
        raise TypeError(f"dims must be a PatchDims, got {type(dims).__name__}")
    b = _int3(block_dims, "block_dims")
    if min(b) < 1:
        raise ValueError(f"block_dims must be positive, got {b}")
    counts = tuple(-(-n // s) for n, s in zip(dims.shape, b))
    axes = [[(i * s, min(s, n - i * s)) for i in range(c)] for n, s, c in zip(dims.shape, b, counts)]
    ranges = tuple(
        BlockRange((x[0], y[0], z[0]), (x[1], y[1], z[1]))
        for z in axes[2]
        for y in axes[1]
        for x in axes[0]
    )
    return BlockDecomposition(block_dims=b, counts=counts, ranges=ranges)


@dataclass(frozen=True)
class InterfaceCopy:
    """Directed ghost fill src interior layer -> dst ghost layer (grid.py:333-352)."""

    src: int
    dst: int
    src_lo: tuple
    dst_lo: tuple
    extent: tuple

    def __post_init__(self):
        for name in ("src_lo", "dst_lo", "extent"):
            object.__setattr__(self, name, _int3(getattr(self, name), name))

    def _desc(self):
        c = _lib.CopyDesc()
        c.src, c.dst = self.src, self.dst
        for a in range(3):
            c.src_lo[a] = self.src_lo[a]
            c.dst_lo[a] = self.dst_lo[a]
            c.extent[a] = self.extent[a]
        return c


def _ghost_axis(copy, patches):
    shape = patches[copy.dst].dims.shape
    axes = [a for a in range(3) if copy.dst_lo[a] in (-1, shape[a])]
    if len(axes) != 1:
        raise ValueError(f"interface copy must target exactly one ghost face, got {copy}")
    return axes[0]


def _reverse(copy, patches):
    """The opposite-direction copy of the same face abutment (grid.py:355-381)."""
    axis = _ghost_axis(copy, patches)
    src_lo, dst_lo = list(copy.dst_lo), list(copy.src_lo)
    if copy.dst_lo[axis] == -1:
        src_lo[axis], dst_lo[axis] = 0, patches[copy.src].dims.shape[axis]
    else:
        src_lo[axis], dst_lo[axis] = patches[copy.dst].dims.shape[axis] - 1, -1
    return InterfaceCopy(copy.dst, copy.src, tuple(src_lo), tuple(dst_lo), copy.extent)


def _overlap(a, b):
    lo, hi = max(a[0], b[0]), min(a[1], b[1])
    return (lo, hi) if lo < hi else None


def _abutments(patches):
    """Face abutments from origins (grid.py:429-465): for every pair, every
    axis on which the boxes touch while overlapping on the other two axes
    yields a forward copy (low patch's last layer -> high patch's low ghost)
    followed by its reverse."""
    out = []
    for ia, ib in itertools.combinations(range(len(patches)), 2):
        ba, bb = patches[ia].global_box, patches[ib].global_box
        ov = [_overlap(x, y) for x, y in zip(ba, bb)]
        if all(o is not None for o in ov):
            raise ValueError(f"patches {ia} and {ib} overlap in the index space")
        for axis in range(3):
            others = [a for a in range(3) if a != axis]
            if any(ov[a] is None for a in others):
                continue
            if ba[axis][1] == bb[axis][0]:
                lo_i, hi_i = ia, ib
            elif bb[axis][1] == ba[axis][0]:
                lo_i, hi_i = ib, ia
            else:
                continue
            low, high = patches[lo_i], patches[hi_i]
            src, dst, ext = [0, 0, 0], [0, 0, 0], [0, 0, 0]
            src[axis], dst[axis], ext[axis] = low.dims.shape[axis] - 1, -1, 1
            for a in others:
                t0, t1 = ov[a]
                src[a], dst[a], ext[a] = t0 - low.origin[a], t0 - high.origin[a], t1 - t0
            fwd = InterfaceCopy(lo_i, hi_i, tuple(src), tuple(dst), tuple(ext))
            out.extend((fwd, _reverse(fwd, patches)))
    return out


def _validate(patches, adjacency):
    """Explicit adjacency lists must be consistent and symmetric (grid.py:384-422)."""
    seen = set(adjacency)
    for c in adjacency:
        if not (0 <= c.src < len(patches) and 0 <= c.dst < len(patches)):
            raise ValueError(f"interface copy references unknown patch: {c}")
        if c.src == c.dst:
            raise ValueError(f"patch cannot abut itself: {c}")
        axis = _ghost_axis(c, patches)
        if c.extent[axis] != 1:
            raise ValueError(f"ghost layer must be one cell thick: {c}")
        s_shape, d_shape = patches[c.src].dims.shape, patches[c.dst].dims.shape
        for a in range(3):
            if c.src_lo[a] < 0 or c.src_lo[a] + c.extent[a] > s_shape[a]:
                raise ValueError(f"source range leaves the interior: {c}")
            if a != axis and (c.dst_lo[a] < 0 or c.dst_lo[a] + c.extent[a] > d_shape[a]):
                raise ValueError(f"ghost range leaves the face: {c}")
        sg = tuple(o + l for o, l in zip(patches[c.src].origin, c.src_lo))
        dg = tuple(o + l for o, l in zip(patches[c.dst].origin, c.dst_lo))
        if sg != dg:
            raise ValueError(f"interface copy is not aligned in the shared index space: {c}")
    for c in adjacency:
        if _reverse(c, patches) not in seen:
            raise ValueError(f"adjacency is not symmetric: no mirror for {c}")


class Level:
    """Non-overlapping patches plus face-abutment adjacency (grid.py:468-520).

    Device plans (patch tables, copy lists, factor bindings) are cached on the
    level; they hold raw pointers into the patches' tensors, which the level
    keeps alive.
    """

    def __init__(self, patches, adjacency=None):
        patches = tuple(patches)
        if not patches:
            raise ValueError("a level needs at least one patch")
        for p in patches:
            if not isinstance(p, Patch):
                raise TypeError(f"level entries must be Patch, got {type(p).__name__}")
        if adjacency is None:
            adjacency = _abutments(patches)
        else:
            adjacency = list(adjacency)
            for ia, ib in itertools.combinations(range(len(patches)), 2):
                ov = [_overlap(x, y) for x, y in zip(patches[ia].global_box, patches[ib].global_box)]
                if all(o is not None for o in ov):
                    raise ValueError(f"patches {ia} and {ib} overlap in the index space")
            _validate(patches, adjacency)
        self.patches = patches
        self.adjacency = tuple(adjacency)
        self._plans = {}

    @property
    def interior_cells(self):
        return sum(p.dims.interior_cells for p in self.patches)

    @property
    def allocated_cells(self):
        return sum(2 * p.dims.total_cells + p.dims.interior_cells for p in self.patches)

    @property
    def device(self):
        devs = {p.device for p in self.patches}
        if len(devs) != 1:
            raise ValueError(f"all patches of a level must share one device, got {devs}")
        return devs.pop()

    def _active(self):
        return bytes(p._active for p in self.patches)

    def _device_plan(self, kind=0, stencil=None, factors=None):
        """The cached libpsmooth plan for (block kind, stencil, factors)."""
        from .stencil import Stencil7

        stencil = stencil if stencil is not None else Stencil7()
        fkey = tuple(id(f) for f in factors) if factors else ()
        key = (kind, stencil, fkey)
        plan = self._plans.get(key)
        if plan is None:
            plan = _DevicePlan(self, kind, stencil, factors)
            self._plans[key] = plan
        return plan

    def refresh_ghosts(self):
        """Physical fill then interface exchange (grid.py:507-517), on device."""
        self._device_plan().refresh(_lib.GHOST_ALL)
        return self

    def __repr__(self):
        return f"Level({len(self.patches)} patches, {len(self.adjacency)} interface copies)"


def _require_cuda(level):
    dev = level.device
    if dev.type != "cuda":
        raise RuntimeError(
            "paper_1208_1975_b200 computes on CUDA only; this level lives on "
            f"{dev} (there is no CPU fallback)"
        )
    for p in level.patches:
        if p.dims.ghost_width != 1:
            raise ValueError("smoothing and ghost exchange require ghost_width == 1")
    return dev


class _DevicePlan:
    """Owner of one psm_plan handle (include/psmooth.h)."""

    def __init__(self, level, kind, stencil, factors):
        self.device = _require_cuda(level)
        lib = _lib.load()
        n = len(level.patches)
        self._level_patches = level.patches  # keep tensors alive
        self._factors = factors  # keep factor handles alive
        pd = (_lib.PatchDesc * n)(*[p._desc() for p in level.patches])
        nc = len(level.adjacency)
        cd = (_lib.CopyDesc * max(1, nc))(*[c._desc() for c in level.adjacency])
        st = stencil._cstruct()
        kname = {_lib.BLOCK_LINE: "line", _lib.BLOCK_PLANE: "plane", _lib.BLOCK_BOX: "box"}.get(kind)
        fac = (ctypes.c_void_p * n)(*[f.handle_for(kname) for f in factors]) if factors else None
        handle = ctypes.c_void_p()
        with torch.cuda.device(self.device):
            _lib.check(lib.psm_plan_create(pd, n, cd, nc, ctypes.byref(st), kind, fac, ctypes.byref(handle)),
                       "psm_plan_create")
        self.handle = handle.value
        self.kind = kind
        self.nplanes = sum(p.dims.nz for p in level.patches)
        self._level = level
        self._slots = 0

    def __del__(self):
        h = getattr(self, "handle", None)
        if h:
            try:
                _lib.load().psm_plan_destroy(h)
            except Exception:
                pass
            self.handle = None

    def _stream(self):
        return ctypes.c_void_p(torch.cuda.current_stream(self.device).cuda_stream)

    def _act(self):
        flags = self._level._active()
        return (ctypes.c_ubyte * len(flags)).from_buffer_copy(flags)

    def reserve(self, slots):
        if slots > self._slots:
            _lib.check(_lib.load().psm_plan_reserve_history(self.handle, slots), "reserve_history")
            self._slots = slots

    def refresh(self, what=_lib.GHOST_ALL):
        with torch.cuda.device(self.device):
            _lib.check(_lib.load().psm_refresh_ghosts(self.handle, self._act(), int(what), self._stream()),
                       "refresh_ghosts")

    def residual(self, slot):
        with torch.cuda.device(self.device):
            _lib.check(_lib.load().psm_residual(self.handle, self._act(), slot, self._stream()), "residual")

    def jacobi(self, omega, slot):
        with torch.cuda.device(self.device):
            _lib.check(_lib.load().psm_jacobi_sweep(self.handle, self._act(), float(omega), slot, self._stream()),
                       "jacobi_sweep")

    def gs(self, omega, mode):
        with torch.cuda.device(self.device):
            _lib.check(_lib.load().psm_gs_sweep(self.handle, self._act(), float(omega), mode, self._stream()),
                       "gs_sweep")

    def sumsq(self, nslots):
        out = (ctypes.c_double * max(1, nslots))()
        with torch.cuda.device(self.device):
            _lib.check(_lib.load().psm_history_sumsq(self.handle, nslots, out, self._stream()), "history")
        return [out[i] for i in range(nslots)]

    def plane_sums(self, slot, out_tensor):
        with torch.cuda.device(self.device):
            _lib.check(_lib.load().psm_history_planes(self.handle, slot, ctypes.c_void_p(out_tensor.data_ptr()),
                                                      self._stream()), "history_planes")


def fill_physical_ghosts(patch):
    """ghost = -interior, x then y then z, on one patch (grid.py:311-330)."""
    if not isinstance(patch, Patch):
        raise TypeError(f"patch must be a Patch, got {type(patch).__name__}")
    if patch.dims.ghost_width != 1:
        raise ValueError("ghost fill requires ghost_width == 1")
    Level([patch], adjacency=[])._device_plan().refresh(_lib.GHOST_PHYSICAL)
    return patch


def exchange_interface_ghosts(level):
    """Interface copies with snapshot semantics (grid.py:523-547): sources are
    interior cells and targets ghost cells, so one launch is order-free."""
    level._device_plan().refresh(_lib.GHOST_INTERFACE)
    return level
