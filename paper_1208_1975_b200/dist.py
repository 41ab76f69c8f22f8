"""Multi-GPU z-slab decomposition: one process per GPU over torch.distributed.

A uniform nx x ny x nz grid is cut into contiguous z-slabs, one patch per rank
with origin (0, 0, k0).  In reference terms this is a multi-patch ``Level``
whose patches abut along z (``grid.py:429-465``); the only cross-rank
``InterfaceCopy`` entries are the two z-faces of each slab.  The reference's
semantics make the split exact for Jacobi (reference
``test_smoother.py:164-196``): ghosts carry previous-step values, so the
sliced run is bit-identical to the single-patch run, history included,
because per-plane residual partial sums are all-gathered and reduced by the
same fixed tree as on one GPU.  GS on slabs is GS on the split level
(inter-slab coupling lagged to step end, as in the reference).

Per Jacobi step on each rank (line blocks), with the halo overlapped:

  sweep boundary planes (k = 0, nz-1) --event--> comm stream: NCCL send of the
  new boundary planes to the z-neighbours, receive theirs into staging
  | sweep interior planes | swap | physical ghosts | wait comm | unpack the
  received planes' interiors into the z-ghost planes (psm_halo_unpack).

The exchange helpers are device-agnostic (they move tensors with
``torch.distributed``); tests drive them with world_size 2 over gloo on CPU.

Fused halo (``SlabDomain(..., halo="p2p")``, line Jacobi): the neighbours'
buffers are mapped into this process with CUDA IPC and the sweep kernel itself
stores its first / last plane into their ghost planes while it writes them, so
a step is one kernel plus two one-thread flag kernels:

  wait(both neighbours finished step s-1) | sweep (+ peer stores) |
  signal(step s done) | swap | physical ghosts (interface z faces kept)

No staging buffer, no pack/unpack, no NCCL call on the data path.  The flags
are ints in device memory (system-scope release / acquire).
"""

from __future__ import annotations

import ctypes
import math

import torch
import torch.distributed as dist

from . import _lib
from .grid import Level, Patch, PatchDims, _int3

__all__ = ["slab_range", "SlabDomain", "exchange_planes", "gather_plane_sums", "PatchLevelDomain", "peer_halo",
           "jacobi_step_p2p",
           "dist_smooth", "dist_smooth_level"]


def slab_range(nz, world, rank):
    """[k0, k1) of rank's slab: contiguous, sizes differ by at most one."""
    if not 0 <= rank < world:
        raise ValueError(f"rank {rank} outside world {world}")
    if nz < world:
        raise ValueError(f"cannot cut {nz} planes into {world} slabs")
    base, extra = divmod(nz, world)
    k0 = rank * base + min(rank, extra)
    return k0, k0 + base + (rank < extra)


def exchange_planes(send_lo, send_hi, recv_lo, recv_hi, lo_rank, hi_rank, group=None):
    """Send ``send_lo`` to ``lo_rank`` and ``send_hi`` to ``hi_rank``; receive
    into ``recv_lo`` from ``lo_rank`` and ``recv_hi`` from ``hi_rank`` (None
    ranks are skipped).  Returns the list of outstanding requests."""
    if send_lo.is_cuda and dist.get_backend(group) == "gloo":
        # gloo has no device-side point-to-point: stage through host memory
        # (used to run the multi-process path with several ranks on one GPU)
        return _exchange_via_host(send_lo, send_hi, recv_lo, recv_hi, lo_rank, hi_rank, group)
    ops = []
    if lo_rank is not None:
        ops.append(dist.P2POp(dist.isend, send_lo, lo_rank, group))
        ops.append(dist.P2POp(dist.irecv, recv_lo, lo_rank, group))
    if hi_rank is not None:
        ops.append(dist.P2POp(dist.isend, send_hi, hi_rank, group))
        ops.append(dist.P2POp(dist.irecv, recv_hi, hi_rank, group))
    if not ops:
        return []
    return dist.batch_isend_irecv(ops)


def _exchange_via_host(send_lo, send_hi, recv_lo, recv_hi, lo_rank, hi_rank, group):
    hs = {k: t.detach().cpu() for k, t in (("lo", send_lo), ("hi", send_hi))}
    hr = {"lo": torch.empty(recv_lo.shape, dtype=recv_lo.dtype), "hi": torch.empty(recv_hi.shape, dtype=recv_hi.dtype)}
    ops = []
    if lo_rank is not None:
        ops.append(dist.P2POp(dist.isend, hs["lo"], lo_rank, group))
        ops.append(dist.P2POp(dist.irecv, hr["lo"], lo_rank, group))
    if hi_rank is not None:
        ops.append(dist.P2POp(dist.isend, hs["hi"], hi_rank, group))
        ops.append(dist.P2POp(dist.irecv, hr["hi"], hi_rank, group))
    for r in dist.batch_isend_irecv(ops) if ops else []:
        r.wait()
    if lo_rank is not None:
        recv_lo.copy_(hr["lo"])
    if hi_rank is not None:
        recv_hi.copy_(hr["hi"])
    return []


def gather_plane_sums(local, group=None):
    """All-gather per-plane vectors (slots, nz_local) in rank order ->
    (slots, sum of nz_local).  Ragged slabs (nz not divisible by the rank
    count) are padded for the collective and cut back after it."""
    world = dist.get_world_size(group)
    n = local.shape[-1]
    sizes = [torch.empty(1, dtype=torch.int64, device=local.device) for _ in range(world)]
    dist.all_gather(sizes, torch.tensor([n], dtype=torch.int64, device=local.device), group=group)
    sizes = [int(t.item()) for t in sizes]
    m = max(sizes)
    padded = local.new_zeros(local.shape[:-1] + (m,))
    padded[..., :n] = local
    parts = [torch.empty_like(padded) for _ in range(world)]
    dist.all_gather(parts, padded, group=group)
    return torch.cat([t[..., :k] for t, k in zip(parts, sizes)], dim=-1)


class SlabDomain:
    """This rank's slab of a global grid plus its z-neighbours."""

    def __init__(self, global_shape, rank=None, world=None, device=None, group=None, halo="nccl"):
        if halo not in ("nccl", "p2p"):
            raise ValueError(f"halo must be 'nccl' or 'p2p', got {halo!r}")
        self.halo = halo
        self._peer = None  # _PeerHalo, set up on the first p2p run
        self.global_shape = _int3(global_shape, "global_shape")
        self.rank = dist.get_rank(group) if rank is None else rank
        self.world = dist.get_world_size(group) if world is None else world
        self.group = group
        nx, ny, nz = self.global_shape
        self.k0, self.k1 = slab_range(nz, self.world, self.rank)
        self.patch = Patch(PatchDims(nx, ny, self.k1 - self.k0), origin=(0, 0, self.k0), device=device)
        # a one-patch level: every face of the slab is physical locally; the
        # cross-rank z faces are overwritten by the exchange (physical first,
        # interface second, as grid.py:507-517)
        self.level = Level([self.patch])
        self.lo_rank = self.rank - 1 if self.rank > 0 else None
        self.hi_rank = self.rank + 1 if self.rank < self.world - 1 else None
        px, py = nx + 2, ny + 2
        dev = self.patch.device
        self.stage_lo = torch.zeros((py, px), dtype=torch.float64, device=dev)
        self.stage_hi = torch.zeros((py, px), dtype=torch.float64, device=dev)
        self._comm_stream = torch.cuda.Stream(dev) if dev.type == "cuda" else None

    @property
    def nz_local(self):
        return self.k1 - self.k0

    def boundary_planes(self, buf_index):
        """Contiguous padded planes k = 0 and k = nz_local-1 of buffer ``buf_index``."""
        b = self.patch._bufs[buf_index]
        return b[1], b[self.nz_local]

    def start_exchange(self, buf_index):
        """Send the boundary planes of buffer ``buf_index`` to the neighbours
        and receive theirs into the staging planes (on the comm stream when
        on CUDA).  Returns the requests; call ``finish_exchange`` after."""
        lo, hi = self.boundary_planes(buf_index)
        if self._comm_stream is None:
            return exchange_planes(lo, hi, self.stage_lo, self.stage_hi, self.lo_rank, self.hi_rank, self.group)
        main = torch.cuda.current_stream(self.patch.device)
        self._comm_stream.wait_stream(main)
        with torch.cuda.stream(self._comm_stream):
            reqs = exchange_planes(lo, hi, self.stage_lo, self.stage_hi, self.lo_rank, self.hi_rank, self.group)
            for r in reqs:
                r.wait()
        return reqs

    def finish_exchange(self, reqs):
        if self._comm_stream is None:
            for r in reqs:
                r.wait()
            return
        torch.cuda.current_stream(self.patch.device).wait_stream(self._comm_stream)

    def unpack(self, plan):
        """Received planes -> z-ghost planes of the active buffer (device)."""
        lib = _lib.load()
        act = (ctypes.c_ubyte * 1)(self.patch._active)
        stream = ctypes.c_void_p(torch.cuda.current_stream(self.patch.device).cuda_stream)
        if self.lo_rank is not None:
            _lib.check(lib.psm_halo_unpack(plan.handle, act, 0, 0, ctypes.c_void_p(self.stage_lo.data_ptr()),
                                           stream), "halo_unpack")
        if self.hi_rank is not None:
            _lib.check(lib.psm_halo_unpack(plan.handle, act, 0, 1, ctypes.c_void_p(self.stage_hi.data_ptr()),
                                           stream), "halo_unpack")


class _PeerHalo:
    """The fused-halo state of one slab: IPC mappings of the z-neighbours'
    buffers and step flags, bound into the device plan."""

    def __init__(self, domain, dp):
        lib = _lib.load()
        p = domain.patch
        # flags[0] is written by the neighbour below, flags[1] by the one above
        self.flags = torch.empty(2, dtype=torch.int32, device=p.device)
        # every rank's earlier signals have landed before any flag is zeroed
        torch.cuda.synchronize(p.device)
        dist.barrier(group=domain.group)
        self.flags.zero_()
        torch.cuda.synchronize(p.device)
        try:
            mine = {"bufs": [_ipc_export(b) for b in p._bufs], "flags": _ipc_export(self.flags),
                    "nz": domain.nz_local, "pci": _pci_bus_id()}
        except (_lib.LibraryError, ValueError) as e:  # still join the gather, so no rank hangs in it
            mine = {"error": str(e)}
        allinfo = [None] * domain.world
        dist.all_gather_object(allinfo, mine, group=domain.group)
        bad = [f"rank {r}: {i['error']}" for r, i in enumerate(allinfo) if "error" in i]
        if bad:
            raise _lib.LibraryError("fused halo: cannot export device buffers (" + "; ".join(bad) + ")")
        self.peer_flags = [None, None]  # the flag word this rank writes in each neighbour
        err = ""
        try:
            for side, r in ((0, domain.lo_rank), (1, domain.hi_rank)):
                if r is None:
                    continue
                info = allinfo[r]
                _require_peer_access(info["pci"], r)
                bufs = [_ipc_import(h, off) for h, off in info["bufs"]]
                flags = _ipc_import(*info["flags"])
                # below: we are its upper neighbour (its flags[1]); above: its flags[0]
                self.peer_flags[side] = flags + (4 if side == 0 else 0)
                _lib.check(lib.psm_plan_set_peer_halo(dp.handle, 0, side, ctypes.c_void_p(bufs[0]),
                                                      ctypes.c_void_p(bufs[1]), int(info["nz"])), "set_peer_halo")
        except (_lib.LibraryError, ValueError) as e:
            err = str(e)
        errs = [None] * domain.world
        dist.all_gather_object(errs, err, group=domain.group)
        if any(errs):
            for side in (0, 1):
                lib.psm_plan_set_peer_halo(dp.handle, 0, side, None, None, 0)
            raise _lib.LibraryError("fused halo unavailable: " + "; ".join(
                f"rank {r}: {e}" for r, e in enumerate(errs) if e))
        base = self.flags.data_ptr()
        if domain.lo_rank is not None and domain.hi_rank is not None:
            self.wait_ptr, self.nwait = base, 2
        elif domain.lo_rank is not None:
            self.wait_ptr, self.nwait = base, 1
        else:
            self.wait_ptr, self.nwait = base + 4, 1
        self.epoch = 0  # flags only grow: value e + s + 1 means step s is done
        self.handle = dp.handle

    def wait(self, value, stream):
        _lib.check(_lib.load().psm_halo_wait(ctypes.c_void_p(self.wait_ptr), self.nwait, int(value), stream),
                   "halo_wait")

    def signal(self, value, stream):
        a, b = self.peer_flags
        _lib.check(_lib.load().psm_halo_signal(ctypes.c_void_p(a), ctypes.c_void_p(b), int(value), stream),
                   "halo_signal")


def _pci_bus_id():
    buf = ctypes.create_string_buffer(32)
    _lib.check(_lib.load().psm_device_pci_bus_id(buf, 32), "device_pci_bus_id")
    return buf.value.decode()


def _require_peer_access(pci, rank):
    """Raise LibraryError unless this process's device can map rank's
    device memory (same device, or cudaDeviceCanAccessPeer)."""
    ok = ctypes.c_int()
    _lib.check(_lib.load().psm_peer_access(pci.encode(), ctypes.byref(ok)), "peer_access")
    if not ok.value:
        raise _lib.LibraryError(f"no peer access from this device to rank {rank}'s device {pci}")


def _ipc_export(t):
    lib = _lib.load()
    h = (ctypes.c_char * 64)()
    off = ctypes.c_longlong()
    _lib.check(lib.psm_ipc_get_handle(ctypes.c_void_p(t.data_ptr()), h, ctypes.byref(off)), "ipc_get_handle")
    return bytes(h), off.value


def _ipc_import(handle, offset):
    lib = _lib.load()
    ptr = ctypes.c_void_p()
    _lib.check(lib.psm_ipc_open_handle(ctypes.c_char_p(handle), int(offset), ctypes.byref(ptr)), "ipc_open_handle")
    return ptr.value


def peer_halo(domain, dp):
    """The domain's fused-halo state bound to device plan ``dp`` (created,
    and the IPC handles exchanged, on first use; collective)."""
    if domain._peer is None or domain._peer.handle != dp.handle:
        domain._peer = _PeerHalo(domain, dp)
    return domain._peer


def _timed(waits, device, fn):
    """Run fn(); with a ``waits`` list, append the (start, end) CUDA events
    bracketing the work it queues on the current stream."""
    if waits is None:
        return fn()
    st = torch.cuda.current_stream(device)
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record(st)
    out = fn()
    b.record(st)
    waits.append((a, b))
    return out


def jacobi_step_p2p(domain, dp, omega, slot, halo, step, events=None, waits=None):
    """One line-Jacobi step of a slab with the fused peer-memory halo (see
    the module docstring).  ``step`` counts from 0 within the current run.
    ``waits``: optional list collecting the CUDA-event pair around the wait
    for the neighbours' previous step (the halo stall of this rank)."""
    p = domain.patch
    stream = ctypes.c_void_p(torch.cuda.current_stream(p.device).cuda_stream)
    _timed(waits, p.device, lambda: halo.wait(halo.epoch + step, stream))
    if events is not None:
        a = torch.cuda.Event(enable_timing=True)
        a.record(torch.cuda.current_stream(p.device))
    dp.jacobi(omega, slot)
    if events is not None:
        b = torch.cuda.Event(enable_timing=True)
        b.record(torch.cuda.current_stream(p.device))
        events.append([(a, b)])
    halo.signal(halo.epoch + step + 1, stream)
    p.swap_buffers()
    dp.refresh(_lib.GHOST_ALL | _lib.GHOST_SKIP_X)


def dist_smooth(domain, config, cache, record_history=True):
    """``smooth`` on a z-slab decomposed grid: every rank calls it with its
    own ``SlabDomain``; returns the (global) history on every rank."""
    from .smoother import _Plan, _gs_mode

    level = domain.level
    plan = _Plan(level, config, cache)
    dp = plan.dev
    lib = _lib.load()
    steps = config.steps
    nzl = domain.nz_local
    fused = domain.halo == "p2p" and config.scheme == "block_jacobi" and plan.kind == "line" and domain.world > 1
    with torch.cuda.device(plan.device):
        halo = None
        if fused:
            try:  # collective; raises on every rank alike
                halo = peer_halo(domain, dp)
            except _lib.LibraryError:
                fused = False  # this plan cannot take the fused halo: NCCL overlap
        dp.reserve(steps + 1)
        dp.refresh(_lib.GHOST_ALL)
        reqs = domain.start_exchange(domain.patch._active)
        domain.finish_exchange(reqs)
        domain.unpack(dp)
        if fused:
            torch.cuda.synchronize(plan.device)
            dist.barrier(group=domain.group)
            stream = ctypes.c_void_p(torch.cuda.current_stream(plan.device).cuda_stream)
            for s in range(steps):
                jacobi_step_p2p(domain, dp, config.omega, s, halo, s)
            halo.wait(halo.epoch + steps, stream)  # the neighbours' last planes are in
            halo.epoch += steps
            dp.residual(steps)
        elif config.scheme == "block_jacobi" and plan.kind == "line":
            for s in range(steps):
                jacobi_step_overlapped(domain, dp, config.omega, s)
            dp.residual(steps)
        else:
            mode = _gs_mode(config)
            if config.scheme != "block_jacobi":
                dp.residual(0)
            for s in range(steps):
                if config.scheme == "block_jacobi":
                    dp.jacobi(config.omega, s)
                    domain.patch.swap_buffers()
                    dp.refresh(_lib.GHOST_ALL | _lib.GHOST_SKIP_X)
                else:
                    dp.gs(config.omega, mode)
                    dp.refresh(_lib.GHOST_ALL | _lib.GHOST_SKIP_X)  # what the sweep left
                reqs = domain.start_exchange(domain.patch._active)
                domain.finish_exchange(reqs)
                domain.unpack(dp)
                if config.scheme != "block_jacobi":
                    dp.residual(s + 1)
            if config.scheme == "block_jacobi":
                dp.residual(steps)
        if not record_history:
            return None
        planes = torch.empty((steps + 1, nzl), dtype=torch.float64, device=plan.device)
        for s in range(steps + 1):
            dp.plane_sums(s, planes[s])
        full = gather_plane_sums(planes, domain.group)
        out = torch.empty(steps + 1, dtype=torch.float64, device=plan.device)
        stream = ctypes.c_void_p(torch.cuda.current_stream(plan.device).cuda_stream)
        for s in range(steps + 1):
            row = full[s].contiguous()
            _lib.check(lib.psm_tree_sum(ctypes.c_void_p(row.data_ptr()), row.numel(),
                                        ctypes.c_void_p(out[s:].data_ptr()), stream), "tree_sum")
        return [math.sqrt(v) for v in out.cpu().tolist()]


def jacobi_step_overlapped(domain, dp, omega, slot, events=None, waits=None):
    """One line-Jacobi step of a slab with the halo exchange overlapped with
    the interior sweep (see the module docstring).  ``events``: optional list
    collecting one list of (start, end) CUDA-event pairs per step, around the
    sweep launches only (kernel time, not the halo); ``waits``: the event
    pair around the compute stream's wait for the exchange and the unpack."""
    lib = _lib.load()
    p = domain.patch
    nzl = domain.nz_local
    act = (ctypes.c_ubyte * 1)(p._active)
    stream = ctypes.c_void_p(torch.cuda.current_stream(p.device).cuda_stream)

    pairs = [] if events is not None else None
    if events is not None:
        events.append(pairs)

    def sweep(k0, k1):
        if k1 > k0:
            if pairs is not None:
                a = torch.cuda.Event(enable_timing=True)
                a.record(torch.cuda.current_stream(p.device))
            _lib.check(lib.psm_jacobi_sweep_planes(dp.handle, act, float(omega), slot, 0, k0, k1, stream),
                       "jacobi_sweep_planes")
            if pairs is not None:
                b = torch.cuda.Event(enable_timing=True)
                b.record(torch.cuda.current_stream(p.device))
                pairs.append((a, b))

    if domain.world == 1:
        sweep(0, nzl)
        p.swap_buffers()
        dp.refresh(_lib.GHOST_ALL | _lib.GHOST_SKIP_X)
        return
    sweep(0, 1)
    sweep(nzl - 1, nzl) if nzl > 1 else None
    new = 1 - p._active  # the buffer the sweep writes
    reqs = domain.start_exchange(new)
    sweep(1, nzl - 1)
    p.swap_buffers()
    dp.refresh(_lib.GHOST_ALL | _lib.GHOST_SKIP_X)

    def land():
        domain.finish_exchange(reqs)
        domain.unpack(dp)

    _timed(waits, p.device, land)


# ---------------------------------------------------------------------------
# Multi-patch levels across GPUs: patches are independent
# within a step, so partition_patches (runtime.py:92-131) assigns them to
# ranks; interface copies between patches of one rank run in the device
# ghost refresh, copies between ranks are packed, sent, received and
# unpacked after it (physical ghosts first, interfaces second, as
# grid.py:507-517).
# ---------------------------------------------------------------------------
class _PatchSpec:
    """A patch description without buffers (for the global adjacency)."""

    def __init__(self, dims, origin):
        self.dims = dims if isinstance(dims, PatchDims) else PatchDims(*_int3(dims, "dims"))
        self.origin = _int3(origin, "origin")

    @property
    def global_box(self):
        return tuple((o, o + n) for o, n in zip(self.origin, self.dims.shape))


class _SpecLevel:
    def __init__(self, specs):
        self.patches = specs


class PatchLevelDomain:
    """This rank's share of a multi-patch level.

    ``specs``: list of (dims, origin) for every patch of the global level, in
    global order.  ``owner[g]`` is the rank of global patch g (greedy cell
    balance by default); ``mine`` the global indices owned here, ascending;
    ``level`` a Level of the owned patches with the interface copies among
    them; ``sends`` / ``recvs`` the cross-rank copies touching this rank."""

    def __init__(self, specs, rank, world, device=None, group=None, assignment="greedy", halo="nccl"):
        from .grid import _abutments
        from .runtime import partition_patches

        if halo not in ("nccl", "p2p"):
            raise ValueError(f"halo must be 'nccl' or 'p2p', got {halo!r}")
        self.halo = halo
        self._peer = None  # _PeerLevelHalo, built on the first p2p run

        self.specs = [_PatchSpec(d, o) for d, o in specs]
        self.rank, self.world, self.group = rank, world, group
        self.adjacency = _abutments(self.specs)
        buckets = partition_patches(_SpecLevel(self.specs), world, assignment)
        self.owner = {g: r for r, b in enumerate(buckets) for g in b}
        self.mine = sorted(g for g, r in self.owner.items() if r == rank)
        if not self.mine:
            raise ValueError(f"rank {rank} owns no patch ({len(self.specs)} patches over {world} ranks)")
        local = {g: i for i, g in enumerate(self.mine)}
        self.local_index = local
        self.patches = [Patch(self.specs[g].dims, self.specs[g].origin, device=device) for g in self.mine]
        from .grid import InterfaceCopy

        inner = [InterfaceCopy(local[c.src], local[c.dst], c.src_lo, c.dst_lo, c.extent)
                 for c in self.adjacency if c.src in local and c.dst in local]
        self.level = Level(self.patches, adjacency=inner)
        # cross-rank copies, in global adjacency order (both sides agree)
        self.sends = [c for c in self.adjacency if c.src in local and c.dst not in local]
        self.recvs = [c for c in self.adjacency if c.dst in local and c.src not in local]

    def _src_view(self, c):
        p = self.patches[self.local_index[c.src]]
        sl = tuple(slice(1 + lo, 1 + lo + e) for lo, e in zip(c.src_lo, c.extent))
        return p.u[sl]

    def _dst_view(self, c):
        p = self.patches[self.local_index[c.dst]]
        sl = tuple(slice(1 + lo, 1 + lo + e) for lo, e in zip(c.dst_lo, c.extent))
        return p.u[sl]

    def exchange(self):
        """Cross-rank interface copies of the active buffers: pack the source
        interior layers, send/receive (grouped), unpack into the ghosts."""
        if self.world == 1:
            return
        out = [self._src_view(c).contiguous() for c in self.sends]
        inb = [torch.empty(tuple(c.extent), dtype=torch.float64, device=self.patches[0].device) for c in self.recvs]
        gloo = out and out[0].is_cuda and dist.get_backend(self.group) == "gloo" or (
            inb and inb[0].is_cuda and dist.get_backend(self.group) == "gloo")
        if gloo:  # host-staged (several ranks on one GPU)
            out_h = [t.cpu() for t in out]
            in_h = [torch.empty(t.shape, dtype=t.dtype) for t in inb]
        else:
            out_h, in_h = out, inb
        ops = [dist.P2POp(dist.isend, t, self.owner[c.dst], self.group) for t, c in zip(out_h, self.sends)]
        ops += [dist.P2POp(dist.irecv, t, self.owner[c.src], self.group) for t, c in zip(in_h, self.recvs)]
        if ops:
            for r in dist.batch_isend_irecv(ops):
                r.wait()
        for c, t in zip(self.recvs, in_h):
            self._dst_view(c).copy_(t)

    def plane_slots(self):
        """(global plane offset, nz) of every owned patch (global patch order)."""
        off, acc = {}, 0
        for g, s in enumerate(self.specs):
            off[g] = acc
            acc += s.dims.nz
        return [(off[g], self.specs[g].dims.nz) for g in self.mine], acc


_NO_PEER = 2**31 - 1  # flag value of ranks that never signal this one


class _PeerLevelHalo:
    """Cross-rank interface copies over peer memory for a PatchLevelDomain.

    Every rank maps the buffers of the remote patches it copies from (CUDA
    IPC) and runs those copies itself, as ordinary interface copies of a
    ghost-only device plan whose patch table holds its own patches followed by
    the mapped remote ones: one launch pulls every cross-rank face straight
    out of the neighbours' memory, no pack, send, receive or unpack.

    Two step flags per rank pair keep the buffers consistent (values only
    grow; e is the epoch of earlier runs):
      ready[q] = e+s+1  producer q swept step s (its new buffer is final)
      read[q]  = e+s+1  consumer q pulled its step-s faces from this rank
    A rank waits ready >= e+s+1 from its producers before pulling, and before
    sweeping step s read >= e+s-1 from its consumers under Jacobi (that sweep
    overwrites the buffer they pulled at step s-2) or read >= e+s under GS
    (in place: the buffer they pulled at step s-1)."""

    def __init__(self, domain, stencil):
        lib = _lib.load()
        dev = domain.patches[0].device
        world, rank = domain.world, domain.rank
        self.producers = sorted({domain.owner[c.src] for c in domain.recvs})
        self.consumers = sorted({domain.owner[c.dst] for c in domain.sends})
        self.ready = torch.empty(world, dtype=torch.int32, device=dev)
        self.read = torch.empty(world, dtype=torch.int32, device=dev)
        torch.cuda.synchronize(dev)
        dist.barrier(group=domain.group)
        init_ready = [0 if q in self.producers else _NO_PEER for q in range(world)]
        init_read = [0 if q in self.consumers else _NO_PEER for q in range(world)]
        self.ready.copy_(torch.tensor(init_ready, dtype=torch.int32))
        self.read.copy_(torch.tensor(init_read, dtype=torch.int32))
        torch.cuda.synchronize(dev)
        try:
            mine = {"patches": {g: [_ipc_export(b) for b in domain.patches[i]._bufs]
                                for i, g in enumerate(domain.mine)},
                    "ready": _ipc_export(self.ready), "read": _ipc_export(self.read), "pci": _pci_bus_id()}
        except (_lib.LibraryError, ValueError) as e:
            mine = {"error": str(e)}
        allinfo = [None] * world
        dist.all_gather_object(allinfo, mine, group=domain.group)
        bad = [f"rank {r}: {i['error']}" for r, i in enumerate(allinfo) if "error" in i]
        if bad:
            raise _lib.LibraryError("peer interface copies: cannot export buffers (" + "; ".join(bad) + ")")
        err = ""
        try:
            # remote source patches, in global order, after the local ones
            remote = sorted({c.src for c in domain.recvs})
            ridx = {g: len(domain.mine) + i for i, g in enumerate(remote)}
            descs = [p._desc() for p in domain.patches]
            self._remote_ptrs = []
            for r in sorted({domain.owner[g] for g in remote} | set(self.consumers) | set(self.producers)):
                if r != rank:
                    _require_peer_access(allinfo[r]["pci"], r)
            for g in remote:
                b0, b1 = (_ipc_import(h, off) for h, off in allinfo[domain.owner[g]]["patches"][g])
                d = _lib.PatchDesc()
                d.buf[0], d.buf[1], d.f = b0, b1, b0  # f is not read by interface copies
                d.nx, d.ny, d.nz = domain.specs[g].dims.shape
                descs.append(d)
                self._remote_ptrs.append((b0, b1))
            copies = []
            for c in domain.recvs:
                cd = _lib.CopyDesc()
                cd.src, cd.dst = ridx[c.src], domain.local_index[c.dst]
                for a in range(3):
                    cd.src_lo[a], cd.dst_lo[a], cd.extent[a] = c.src_lo[a], c.dst_lo[a], c.extent[a]
                copies.append(cd)
            self.nall = len(descs)
            pd = (_lib.PatchDesc * self.nall)(*descs)
            cda = (_lib.CopyDesc * max(1, len(copies)))(*copies)
            st = stencil._cstruct()
            handle = ctypes.c_void_p()
            _lib.check(lib.psm_plan_create(pd, self.nall, cda, len(copies), ctypes.byref(st), 0, None,
                                           ctypes.byref(handle)), "psm_plan_create (peer copies)")
            self.plan = handle.value
            # the flag words this rank writes in each neighbour
            self.ready_out = [_ipc_import(*allinfo[q]["ready"]) + 4 * rank for q in self.consumers]
            self.read_out = [_ipc_import(*allinfo[q]["read"]) + 4 * rank for q in self.producers]
        except (_lib.LibraryError, ValueError) as e:
            err = str(e)
        errs = [None] * world
        dist.all_gather_object(errs, err, group=domain.group)
        if any(errs):
            raise _lib.LibraryError("peer interface copies unavailable: " + "; ".join(
                f"rank {r}: {e}" for r, e in enumerate(errs) if e))
        self.epoch = 0
        self.world = world

    def __del__(self):
        h = getattr(self, "plan", None)
        if h:
            try:
                _lib.load().psm_plan_destroy(h)
            except Exception:
                pass

    def _signal(self, ptrs, value, stream):
        lib = _lib.load()
        for i in range(0, len(ptrs), 2):
            a = ptrs[i]
            b = ptrs[i + 1] if i + 1 < len(ptrs) else None
            _lib.check(lib.psm_halo_signal(ctypes.c_void_p(a), ctypes.c_void_p(b), int(value), stream),
                       "halo_signal")

    def _wait(self, flags, value, stream):
        _lib.check(_lib.load().psm_halo_wait(ctypes.c_void_p(flags.data_ptr()), self.world, int(value), stream),
                   "halo_wait")

    def before_sweep(self, s, in_place, stream):
        lag = 0 if in_place else 1
        if s >= 1 + lag and self.consumers:
            self._wait(self.read, self.epoch + s - lag, stream)

    def after_sweep(self, s, active, stream):
        """The step's sweep, swap and local refresh are queued: publish, pull
        the remote faces into this rank's ghosts, acknowledge."""
        self._signal(self.ready_out, self.epoch + s + 1, stream)
        if self.producers:
            self._wait(self.ready, self.epoch + s + 1, stream)
            act = (ctypes.c_ubyte * self.nall)(*([active] * self.nall))
            _lib.check(_lib.load().psm_refresh_ghosts(self.plan, act, _lib.GHOST_INTERFACE, stream),
                       "peer interface copies")
        self._signal(self.read_out, self.epoch + s + 1, stream)


def dist_smooth_level(domain, config, cache):
    """``smooth`` on a multi-patch level split over ranks by patch: every rank
    calls it with its own ``PatchLevelDomain``; returns the global history on
    every rank (bit-identical to the single-process run: per-plane partial
    sums are reduced in global plane order by the same fixed tree)."""
    from .smoother import _Plan, _gs_mode

    level = domain.level
    plan = _Plan(level, config, cache)
    dp = plan.dev
    lib = _lib.load()
    steps = config.steps
    jac = config.scheme == "block_jacobi"
    with torch.cuda.device(plan.device):
        peer = None
        if domain.halo == "p2p" and domain.world > 1:
            try:  # collective; raises on every rank alike
                if domain._peer is None:
                    domain._peer = _PeerLevelHalo(domain, config.stencil)
                peer = domain._peer
            except _lib.LibraryError:
                peer = None  # NCCL exchange
        stream = ctypes.c_void_p(torch.cuda.current_stream(plan.device).cuda_stream)
        dp.reserve(steps + 1)
        dp.refresh(_lib.GHOST_ALL)
        domain.exchange()
        if peer is not None:
            torch.cuda.synchronize(plan.device)
            dist.barrier(group=domain.group)
        if not jac:
            dp.residual(0)
        mode = _gs_mode(config)
        for s in range(steps):
            if peer is not None:
                peer.before_sweep(s, not jac, stream)
            if jac:
                dp.jacobi(config.omega, s)
                for p in level.patches:
                    p.swap_buffers()
                dp.refresh(_lib.GHOST_ALL | _lib.GHOST_SKIP_X)
            else:
                dp.gs(config.omega, mode)
                dp.refresh(_lib.GHOST_ALL | _lib.GHOST_SKIP_X)  # what the sweep left
            if peer is not None:
                peer.after_sweep(s, level.patches[0]._active, stream)
            else:
                domain.exchange()
            if not jac:
                dp.residual(s + 1)
        if peer is not None:
            peer.epoch += steps
        if jac:
            dp.residual(steps)
        slots, total = domain.plane_slots()
        nloc = sum(n for _, n in slots)
        local = torch.empty((steps + 1, nloc), dtype=torch.float64, device=plan.device)
        for s in range(steps + 1):
            dp.plane_sums(s, local[s])
        full = torch.zeros((steps + 1, total), dtype=torch.float64, device=plan.device)
        c = 0
        for off, n in slots:
            full[:, off:off + n] = local[:, c:c + n]
            c += n
        if domain.world > 1:  # each plane has exactly one owner: the sum is exact
            if full.is_cuda and dist.get_backend(domain.group) == "gloo":
                fh = full.cpu()
                dist.all_reduce(fh, group=domain.group)
                full.copy_(fh)
            else:
                dist.all_reduce(full, group=domain.group)
        out = torch.empty(steps + 1, dtype=torch.float64, device=plan.device)
        stream = ctypes.c_void_p(torch.cuda.current_stream(plan.device).cuda_stream)
        for s in range(steps + 1):
            row = full[s].contiguous()
            _lib.check(lib.psm_tree_sum(ctypes.c_void_p(row.data_ptr()), row.numel(),
                                        ctypes.c_void_p(out[s:].data_ptr()), stream), "tree_sum")
        return [math.sqrt(v) for v in out.cpu().tolist()]
