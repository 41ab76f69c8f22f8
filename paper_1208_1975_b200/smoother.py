"""Block relaxation sweeps on the device (reference ``smoother.py:1-214``).

Same names, signatures, defaults, validation and history semantics as the
reference:

* ``smooth(level, config, cache, timers=None) -> (level, history)`` runs a
  ghost refresh, records ``history[0]``, then ``config.steps`` steps, each
  followed by a refresh and a history entry (``smoother.py:197-214``);
* ``smooth_jacobi_step`` / ``smooth_chaotic_gs_step`` run one step without
  history and without a leading refresh (``smoother.py:172-194``);
* ``residual_norm(level, stencil)`` is the global L2 norm of f - A u.

Every step is one or two stream-ordered ``libpsmooth`` launches: there is no
per-block Python dispatch and no host synchronisation until the history is
read back once at the end.  Jacobi fuses the history into the sweep: sweep s
computes ``r = f - A u^s`` for every cell anyway, so its squared norm is
``history[s]``; only the last entry needs a separate residual pass.

Also exported: the north-star convenience form
``smooth(u, f, sweeps, block='line'|'plane', method='jacobi'|'gs')`` on bare
arrays, which builds a one-patch level and calls the reference form.
"""

from __future__ import annotations

import math
from dataclasses import dataclass, field

import numpy as np
import torch

from . import _lib
from .blocklinalg import InverseCache
from .grid import Level, Patch, PatchDims, _int3, _require_cuda
from .runtime import ExecutionStrategy
from .stencil import Stencil7

__all__ = [
    "SCHEMES",
    "SmootherConfig",
    "smooth",
    "smooth_jacobi_step",
    "smooth_chaotic_gs_step",
    "residual_norm",
    "block_shape_of",
    "block_update",
]

SCHEMES = ("block_jacobi", "chaotic_block_gs")
_DEFAULT_OMEGA = {"block_jacobi": 0.8, "chaotic_block_gs": 1.0}  # smoother.py:51


@dataclass(frozen=True)
class SmootherConfig:
    """What to run: scheme, block shape, damping, steps, dispatch (smoother.py:54-87)."""

    scheme: str
    block_dims: tuple
    omega: float = None
    steps: int = 1
    strategy: ExecutionStrategy = field(default_factory=ExecutionStrategy.serial)
    stencil: Stencil7 = field(default_factory=Stencil7)
    seed: int = 42

    def __post_init__(self):
        if self.scheme not in SCHEMES:
            raise ValueError(f"unknown scheme {self.scheme!r}, expected one of {SCHEMES}")
        object.__setattr__(self, "block_dims", _int3(self.block_dims, "block_dims"))
        if any(b < 1 for b in self.block_dims):
            raise ValueError(f"block_dims must be positive, got {self.block_dims}")
        omega = _DEFAULT_OMEGA[self.scheme] if self.omega is None else self.omega
        omega = float(omega)
        if not 0.0 < omega <= 1.0:
            raise ValueError(f"omega must lie in (0, 1], got {omega}")
        object.__setattr__(self, "omega", omega)
        if not isinstance(self.steps, int) or isinstance(self.steps, bool) or self.steps < 1:
            raise ValueError(f"steps must be a positive integer, got {self.steps!r}")
        if not isinstance(self.strategy, ExecutionStrategy):
            raise TypeError("strategy must be an ExecutionStrategy")
        if not isinstance(self.stencil, Stencil7):
            raise TypeError("stencil must be a Stencil7")
        if not isinstance(self.seed, int) or isinstance(self.seed, bool):
            raise ValueError(f"seed must be an integer, got {self.seed!r}")


def block_shape_of(dims, block_dims):
    """(extent, kind) of the blocks block_dims make on the patch, after the
    reference's truncation (grid.py:298-306): 'line' for one block per x-line
    ((>=nx,1,1)), 'plane' for one per xy-plane ((>=nx,>=ny,1)), 'box' for
    blocks of at most 8 cells per axis (the paper's cubic blocks, truncated at
    the patch edges by the kernel); ValueError otherwise.  A plane block on a
    ny == 1 patch is a line block."""
    b = _int3(block_dims, "block_dims")
    nx, ny, nz = dims.shape
    if b[0] >= nx and b[2] == 1:
        if b[1] == 1 or ny == 1 and b[1] >= 1:
            return (nx, 1, 1), "line"
        if b[1] >= ny:
            return (nx, ny, 1), "plane"
    ext = (min(b[0], nx), min(b[1], ny), min(b[2], nz))
    if max(ext) <= 8:
        return ext, "box"
    raise ValueError(
        f"block_dims {b} on a {dims.shape} patch are neither line blocks (>=nx,1,1), plane blocks "
        "(>=nx,>=ny,1) nor box blocks of at most 8 cells per axis; the device smoother implements exactly those"
    )


class _Plan:
    """Per-level device plan + factor objects (smoother.py:112-124)."""

    def __init__(self, level, config, cache):
        if not isinstance(level, Level):
            raise TypeError(f"level must be a Level, got {type(level).__name__}")
        dev = _require_cuda(level)
        kinds, factors = set(), []
        for p in level.patches:
            ext, kind = block_shape_of(p.dims, config.block_dims)
            kinds.add(kind)
            factors.append(cache.get(config.stencil, ext, dev, kind))
        if len(kinds) != 1:
            raise ValueError(f"block_dims {config.block_dims} make mixed line/plane/box blocks on this level")
        self.kind = kinds.pop()
        ckind = {"line": _lib.BLOCK_LINE, "plane": _lib.BLOCK_PLANE, "box": _lib.BLOCK_BOX}[self.kind]
        self.dev = level._device_plan(ckind, config.stencil, factors)
        self.device = dev


def _gs_mode(config):
    return _lib.GS_CHAOTIC if config.strategy.resolved_gs_mode == "chaotic" else _lib.GS_WAVEFRONT


class _GhostTimer:
    """CUDA-event timing of ghost refreshes for timers['ghost_seconds']."""

    def __init__(self, timers, device):
        self.timers = timers
        self.device = device
        self.pairs = []

    def __enter__(self):
        if self.timers is not None:
            e = torch.cuda.Event(enable_timing=True)
            e.record(torch.cuda.current_stream(self.device))
            self.pairs.append([e, None])
        return self

    def __exit__(self, *exc):
        if self.timers is not None:
            e = torch.cuda.Event(enable_timing=True)
            e.record(torch.cuda.current_stream(self.device))
            self.pairs[-1][1] = e
        return False

    def commit(self):
        if self.timers is None:
            return
        torch.cuda.current_stream(self.device).synchronize()
        secs = sum(a.elapsed_time(b) for a, b in self.pairs) / 1e3
        self.timers["ghost_seconds"] = self.timers.get("ghost_seconds", 0.0) + secs


def _swap_all(level):
    for p in level.patches:
        p.swap_buffers()


def _run(level, config, plan, steps, history, timers):
    """Shared driver: returns the list of squared history entries (or None).

    Without ``timers`` the whole step sequence is one ``psm_smooth_steps``
    call, which replays a captured CUDA graph from the second call with the
    same shape on; with ``timers`` (per-refresh CUDA events) it runs eagerly."""
    if timers is None:
        return _run_graph(level, config, plan, steps, history)
    dp = plan.dev
    gt = _GhostTimer(timers, plan.device)
    with torch.cuda.device(plan.device):
        if history:
            dp.reserve(steps + 1)
            with gt:
                dp.refresh(_lib.GHOST_ALL)
        if config.scheme == "block_jacobi":
            for s in range(steps):
                dp.jacobi(config.omega, s if history else -1)
                _swap_all(level)
                with gt:
                    dp.refresh(_lib.GHOST_ALL | _lib.GHOST_SKIP_X)
            if history:
                dp.residual(steps)
        else:
            mode = _gs_mode(config)
            if history:
                dp.residual(0)
            for s in range(steps):
                dp.gs(config.omega, mode)
                with gt:
                    dp.refresh(_lib.GHOST_ALL | _lib.GHOST_SKIP_X)  # what the sweep left
                if history:
                    dp.residual(s + 1)
        sums = dp.sumsq(steps + 1) if history else None
    gt.commit()
    return sums


def _run_graph(level, config, plan, steps, history):
    dp = plan.dev
    jac = config.scheme == "block_jacobi"
    with torch.cuda.device(plan.device):
        if history:
            dp.reserve(steps + 1)
        act = dp._act()
        _lib.check(_lib.load().psm_smooth_steps(dp.handle, act, 0 if jac else 1, float(config.omega), int(steps),
                                                _gs_mode(config), 1 if history else 0, dp._stream()),
                   "smooth_steps")
        if jac:
            for _ in range(steps):
                _swap_all(level)
        sums = dp.sumsq(steps + 1) if history else None
    return sums


def smooth_jacobi_step(level, config, cache):
    """One damped block Jacobi step; expects ghosts already refreshed
    (smoother.py:172-181)."""
    if config.scheme != "block_jacobi":
        raise ValueError(f"config.scheme is {config.scheme!r}, not block_jacobi")
    _run(level, config, _Plan(level, config, cache), 1, False, None)
    return level


def smooth_chaotic_gs_step(level, config, cache):
    """One block Gauss-Seidel step in place; expects ghosts refreshed
    (smoother.py:184-194)."""
    if config.scheme != "chaotic_block_gs":
        raise ValueError(f"config.scheme is {config.scheme!r}, not chaotic_block_gs")
    _run(level, config, _Plan(level, config, cache), 1, False, None)
    return level


def block_update(u_b, r_b, inv, omega):
    """One exact block relaxation u_b + omega * (inv @ r_b) as a new vector
    (smoother.py:90-93): the reference's ascending-column matvec and its two
    roundings, in one device kernel (psm_matvec); bit-identical."""
    from .blocklinalg import _matvec

    return _matvec(inv, r_b, u_b, omega)


def residual_norm(level, stencil):
    """Global L2 norm of f - A u over all patch interiors (smoother.py:96-109).
    Ghosts are read as stored.  Per-tile partials are summed in a fixed order
    on the device (deterministic; not exactly rounded like math.fsum)."""
    if not isinstance(stencil, Stencil7):
        raise TypeError("stencil must be a Stencil7")
    dev = _require_cuda(level)
    dp = level._device_plan(0, stencil, None)
    with torch.cuda.device(dev):
        dp.reserve(1)
        dp.residual(0)
        return math.sqrt(dp.sumsq(1)[0])


def _smooth_level(level, config, cache, timers=None):
    plan = _Plan(level, config, cache)
    sums = _run(level, config, plan, config.steps, True, timers)
    return level, [math.sqrt(s) for s in sums]


def _smooth_arrays(u, f, sweeps, block="line", method="jacobi", omega=None, strategy=None, stencil=None,
                   device=None):
    """North-star form: smooth the interior field ``u`` (nx,ny,nz) against
    ``f`` on one patch with homogeneous Dirichlet faces.  ``u`` is updated in
    place when it is a tensor or ndarray; returns (u, history)."""
    if block not in ("line", "plane"):
        raise ValueError(f"block must be 'line' or 'plane', got {block!r}")
    if method not in ("jacobi", "gs"):
        raise ValueError(f"method must be 'jacobi' or 'gs', got {method!r}")
    shape = tuple(int(n) for n in u.shape)
    if len(shape) != 3 or tuple(f.shape) != shape:
        raise ValueError(f"u and f must be equal 3-d arrays, got {tuple(u.shape)} and {tuple(f.shape)}")
    dev = torch.device(device) if device is not None else (
        u.device if torch.is_tensor(u) and u.is_cuda else torch.device("cuda", torch.cuda.current_device()))
    p = Patch(PatchDims(*shape), device=dev)
    p.interior[...] = torch.as_tensor(np.asarray(u) if not torch.is_tensor(u) else u, dtype=torch.float64).to(dev)
    p.f[...] = torch.as_tensor(np.asarray(f) if not torch.is_tensor(f) else f, dtype=torch.float64).to(dev)
    level = Level([p])
    bd = (shape[0], 1, 1) if block == "line" else (shape[0], shape[1], 1)
    cfg = SmootherConfig(scheme="block_jacobi" if method == "jacobi" else "chaotic_block_gs", block_dims=bd,
                         omega=omega, steps=int(sweeps),
                         strategy=strategy if strategy is not None else ExecutionStrategy.device(),
                         stencil=stencil if stencil is not None else Stencil7())
    _, hist = _smooth_level(level, cfg, InverseCache())
    out = p.interior
    if torch.is_tensor(u):
        u.copy_(out.to(u.device))
        return u, hist
    if isinstance(u, np.ndarray) and u.flags.writeable:
        u[...] = out.cpu().numpy()
        return u, hist
    return out.clone(), hist


def smooth(level, config=None, cache=None, timers=None, **kw):
    """Run ``config.steps`` smoothing steps and record the residual history
    (smoother.py:197-214); returns (level, history) with the level updated in
    place.  Called as ``smooth(u, f, sweeps, block=..., method=...)`` on bare
    arrays it runs the north-star convenience form instead."""
    if isinstance(level, Level):
        if not isinstance(config, SmootherConfig):
            raise TypeError("config must be a SmootherConfig")
        if cache is None:
            raise TypeError("smooth(level, config, cache) needs an InverseCache")
        return _smooth_level(level, config, cache, timers)
    # north-star form: smooth(u, f, sweeps, block=..., method=...)
    u, f, sweeps = level, config, cache
    if timers is not None:
        kw.setdefault("block", timers)
    return _smooth_arrays(u, f, sweeps, **kw)
