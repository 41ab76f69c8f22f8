#!/usr/bin/env python
"""Benchmark: G unknown-updates/s per fp64 smoothing sweep and % of HBM roofline.

Workload (BASELINE.json configs[4], the one the metric's 1/2/4/8-GPU figure is
quoted on): a 1024^3 uniform grid, line block Jacobi (block_dims (1024,1,1),
omega 0.8), z-slab decomposed over N GPUs (one process per GPU, launched by
torchrun for N > 1); strong scaling, the global grid is fixed.  A step is one
smoother step as the reference runs it (smoother.py:138-153): the line-Jacobi
sweep with its fused residual-norm partials, the buffer swap, the physical
ghost refresh and, for N > 1, the halo: by default fused into the sweep
(PSM_HALO=p2p: the kernel stores its boundary planes straight into the
neighbours' ghost planes over CUDA IPC / NVLink, step flags instead of a
collective), or PSM_HALO=nccl: NCCL send/recv overlapped with the interior
sweep.  p2p falls back to nccl when a rank cannot map its neighbours.

Keys beyond the base contract:
  roofline      dominant kernel (line Jacobi sweep) achieved GB/s from 24
                algorithmic bytes per update (read u, read f, write v) over its
                CUDA-event duration inside the timed region, vs the measured
                copy bandwidth in MEASURED_PEAKS.json
  north_star_512  the BASELINE north-star target: device-timed 512^3
                line-Jacobi sweep and its fraction of 8 TB/s (N=1 only)
  cpu_baseline  the oracle's C restatement (OpenMP, all host cores) on a
                bounded slab of the same workload ("port"), with
                ``reference_py``: the reference package itself (patchsmooth
                from baseline/_ref, serial, its own run_bench) on a smaller
                slab of the same line length
  e2e           the same metric through the public API with host buffers:
                per call H2D of u and f from pinned memory, smooth(...) with
                --e2e-sweeps sweeps including the history, D2H of u + history
`--impl reference` runs only the CPU port on rank 0 (see cpu_baseline).
"""

from __future__ import annotations

import argparse
import ctypes
import json
import math
import os
import statistics
import subprocess
import sys
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)

METRIC = "Gunknown-updates/s per smoothing sweep (fp64) and % of HBM roofline, 1/2/4/8 GPU"
UNIT = "Gupdates/s"
BYTES_PER_UPDATE = 24  # read u 8, read f 8, write v 8
FALLBACK_HBM = 6650.0


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", choices=("ours", "reference"), default="ours")
    ap.add_argument("--shape", type=int, nargs=3, default=(1024, 1024, 1024))
    ap.add_argument("--e2e-sweeps", type=int, default=10)
    ap.add_argument("--e2e-calls", type=int, default=2)
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-north-star", action="store_true")
    ap.add_argument("--cpu-seconds", type=float, default=10.0)
    return ap.parse_args()


# ---------------------------------------------------------------------------
# CPU port (oracle/psm_oracle.c) -- the reference arm and cpu_baseline
# ---------------------------------------------------------------------------
def _oracle_lib():
    path = os.path.join(ROOT, "oracle", "build", "liboracle.so")
    if not os.path.exists(path):
        subprocess.run(["make", "-C", os.path.join(ROOT, "oracle")], check=True, capture_output=True)
    lib = ctypes.CDLL(path)
    lib.oracle_line_jacobi.restype = ctypes.c_double
    lib.oracle_line_jacobi.argtypes = [ctypes.c_void_p] * 3 + [ctypes.c_int] * 3 + [
        ctypes.c_double, ctypes.c_void_p, ctypes.c_double, ctypes.c_int, ctypes.c_int]
    lib.oracle_fill_ghosts.argtypes = [ctypes.c_void_p] + [ctypes.c_int] * 4
    lib.oracle_max_threads.restype = ctypes.c_int
    return lib


class CpuPort:
    """One bounded slab (nx x ny x 8 planes) of the workload on the host."""

    def __init__(self, nx, ny, nz=8):
        import numpy as np

        self.lib = _oracle_lib()
        self.threads = os.cpu_count() or 1
        self.shape = (nx, ny, nz)
        rng = np.random.default_rng(42)
        pad = (nz + 2, ny + 2, nx + 2)
        self.u = np.zeros(pad)
        self.v = np.zeros(pad)
        self.u[1:-1, 1:-1, 1:-1] = rng.random((nz, ny, nx))
        self.f = rng.standard_normal((nz, ny, nx))
        self.faces = (ctypes.c_double * 6)(*([-1.0] * 6))
        self.lib.oracle_fill_ghosts(self.u.ctypes.data, nx, ny, nz, self.threads)

    @property
    def cells(self):
        return self.shape[0] * self.shape[1] * self.shape[2]

    def step(self):
        nx, ny, nz = self.shape
        self.lib.oracle_line_jacobi(self.u.ctypes.data, self.f.ctypes.data, self.v.ctypes.data, nx, ny, nz, 6.0,
                                    self.faces, 0.8, 1, self.threads)
        self.u, self.v = self.v, self.u
        self.lib.oracle_fill_ghosts(self.u.ctypes.data, nx, ny, nz, self.threads)

    def rate(self, seconds=None, steps=None, warmup=1):
        for _ in range(warmup):
            self.step()
        n, t0 = 0, time.perf_counter()
        while True:
            self.step()
            n += 1
            el = time.perf_counter() - t0
            if (steps is not None and n >= steps) or (steps is None and el >= seconds):
                break
        return self.cells * n / el / 1e9, n, el

    def describe(self, value, n, el):
        nx, ny, nz = self.shape
        return {
            "value": value,
            "unit": UNIT,
            "cores": self.threads,
            "kind": "port",
            "sample": f"{n} line-Jacobi sweeps (+ghost fill, fused norm) of a {nx}x{ny}x{nz} slab of the "
                      f"workload ({el:.1f} s), oracle/psm_oracle.c with {self.threads} OpenMP threads",
        }


# ---------------------------------------------------------------------------
# clocks sampled during the timed region
# ---------------------------------------------------------------------------
class ClockSampler:
    FIELDS = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, index):
        self.index = index
        self.proc = None
        self.lines = []

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--query-gpu={self.FIELDS}", "--format=csv,noheader,nounits", "-lms", "100",
                 "-i", str(self.index)], stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
        except OSError:
            self.proc = None
        time.sleep(0.3)
        return self

    def __exit__(self, *exc):
        if self.proc is not None:
            time.sleep(0.2)
            self.proc.terminate()
            out, _ = self.proc.communicate(timeout=10)
            self.lines = [ln for ln in out.splitlines() if ln.strip()]
        return False

    def summary(self):
        sm, mx, reasons = [], None, set()
        names = ("hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap")
        for ln in self.lines:
            parts = [p.strip() for p in ln.split(",")]
            if len(parts) < 9:
                continue
            try:
                sm.append(float(parts[1]))
                mx = float(parts[2])
            except ValueError:
                continue
            for n, flag in zip(names, parts[5:9]):
                if flag.lower() == "active":
                    reasons.add(n)
        if not sm:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"]}
        return {"sm_mhz": statistics.median(sm), "sm_max_mhz": mx, "reasons": sorted(reasons), "samples": len(sm)}


def _peaks():
    path = os.path.join(ROOT, "MEASURED_PEAKS.json")
    try:
        with open(path) as fh:
            d = json.load(fh)
        return float(d["hbm_gbs"]), "MEASURED_PEAKS.json hbm_gbs (measured copy, of measured)"
    except (OSError, KeyError, ValueError):
        return FALLBACK_HBM, "B200_PROFILING.md fallback 6.65 TB/s (of fallback)"


def _traffic(workload_key):
    path = os.path.join(ROOT, "profiles", "ncu_traffic.json")
    try:
        with open(path) as fh:
            return json.load(fh).get(workload_key)
    except (OSError, ValueError):
        return None


# ---------------------------------------------------------------------------
def run_reference(args, rank, world):
    if rank != 0:
        return
    nx, ny, _ = args.shape
    port = CpuPort(nx, ny, 8)
    value, n, el = port.rate(steps=args.steps, warmup=args.warmup)
    cb = port.describe(value, n, el)
    cb["reference_py"] = _reference_py(nx)
    line = {
        "impl": "reference",
        "metric": METRIC,
        "value": value,
        "unit": UNIT,
        "n_gpus": args.gpus,
        "steps": args.steps,
        "warmup": args.warmup,
        "ms_per_step": el / n * 1e3,
        "higher_is_better": True,
        "scaling": "strong",
        "vs_baseline": None,
        "dtype": "f64",
        "data": "synthetic: u0 ~ U[0,1) (default_rng(42)), f ~ N(0,1), host memory",
        "config": {"workload": f"C5 bounded sample: {nx}x{ny}x8 slab of the {args.shape[0]}^3 line-Jacobi grid",
                   "block_dims": [nx, 1, 1], "omega": 0.8},
        "cpu_baseline": cb,
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


def run_ours(args, rank, world, local_rank):
    import torch
    import torch.distributed as dist

    import paper_1208_1975_b200 as ps
    from paper_1208_1975_b200 import _lib
    from paper_1208_1975_b200.dist import SlabDomain, jacobi_step_overlapped, jacobi_step_p2p, peer_halo
    from paper_1208_1975_b200.smoother import _Plan

    dev = torch.device("cuda", local_rank)
    torch.cuda.set_device(dev)
    nx, ny, nz = args.shape
    halo_mode = os.environ.get("PSM_HALO", "p2p")
    dom = SlabDomain((nx, ny, nz), rank, world, device=dev, group=None, halo=halo_mode) if world > 1 else None
    if dom is None:
        # single GPU: the same class without a process group
        dom = SlabDomain((nx, ny, nz), 0, 1, device=dev)
    p = dom.patch
    gen = torch.Generator(device=dev)
    gen.manual_seed(1234 + rank)
    p.interior.copy_(torch.rand(p.interior.shape, generator=gen, device=dev, dtype=torch.float64))
    p.f.copy_(torch.randn(p.f.shape, generator=gen, device=dev, dtype=torch.float64))
    cfg = ps.SmootherConfig(scheme="block_jacobi", block_dims=(nx, 1, 1), omega=0.8, steps=1,
                            strategy=ps.ExecutionStrategy.device(devices=world))
    cache = ps.InverseCache()
    plan = _Plan(dom.level, cfg, cache)
    dp = plan.dev
    dp.reserve(2)
    lib = _lib.load()
    stream = torch.cuda.current_stream(dev)

    def barrier():
        if world > 1:
            dist.barrier()

    halo = None
    if world > 1 and halo_mode == "p2p":
        ok = 1
        try:
            halo = peer_halo(dom, dp)
        except (_lib.LibraryError, ValueError) as e:  # no IPC mapping: every rank falls back to NCCL
            print(f"rank {rank}: fused halo unavailable ({e}); using NCCL", file=sys.stderr)
            ok = 0
        flag = torch.tensor([ok], dtype=torch.int32, device=dev)
        dist.all_reduce(flag, op=dist.ReduceOp.MIN)
        if not int(flag.item()):
            halo = None
            dom.halo = halo_mode = "nccl"
            for side in (0, 1):  # unbind whatever was mapped
                _lib.check(lib.psm_plan_set_peer_halo(dp.handle, 0, side, None, None, 0), "set_peer_halo")
            dom._peer = None

    # initial ghosts (physical + halo)
    dp.refresh(_lib.GHOST_ALL)
    if world > 1:
        dom.finish_exchange(dom.start_exchange(p._active))
        dom.unpack(dp)
        torch.cuda.synchronize(dev)
        dist.barrier()
    nstep = [0]  # p2p: steps since the halo's epoch

    halo_waits = []  # N > 1: per step, the event pair around this rank's halo stall

    def step(s, record):
        # the sweep launches are bracketed by events on the launching stream
        if halo is not None:
            jacobi_step_p2p(dom, dp, cfg.omega, s % 2, halo, nstep[0], events=multi_sweeps if record else None,
                            waits=halo_waits if record else None)
            nstep[0] += 1
        elif world > 1:
            jacobi_step_overlapped(dom, dp, cfg.omega, s % 2, events=multi_sweeps if record else None,
                                   waits=halo_waits if record else None)
        else:
            _single_step(s)

    act_buf = (ctypes.c_ubyte * 1)()
    sweep_only = []
    multi_sweeps = []  # N > 1: per step, the event pairs of the three range sweeps

    def _single_step(s):
        act_buf[0] = p._active
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        _lib.check(lib.psm_jacobi_sweep(dp.handle, act_buf, cfg.omega, s % 2, ctypes.c_void_p(stream.cuda_stream)),
                   "jacobi_sweep")
        e1.record(stream)
        sweep_only.append((e0, e1))
        p.swap_buffers()
        dp.refresh(_lib.GHOST_ALL | _lib.GHOST_SKIP_X)

    for s in range(args.warmup):
        step(s, False)
    sweep_only.clear()
    torch.cuda.synchronize(dev)
    barrier()
    launches0 = lib.psm_plan_launches(dp.handle)
    start = torch.cuda.Event(enable_timing=True)
    stop = torch.cuda.Event(enable_timing=True)
    with ClockSampler(local_rank) as clk:
        barrier()
        torch.cuda.synchronize(dev)
        start.record(stream)
        for s in range(args.steps):
            step(s, True)
        stop.record(stream)
        torch.cuda.synchronize(dev)
        barrier()
    launches = lib.psm_plan_launches(dp.handle) - launches0
    if halo is not None:
        launches += 2 * args.steps  # the flag wait / signal kernels (not counted by the plan)
        halo.epoch += nstep[0]
    ms = start.elapsed_time(stop)
    t = torch.tensor([ms], dtype=torch.float64, device=dev)
    if world > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    ms_total = float(t.item())
    cells = nx * ny * nz
    value = cells * args.steps / (ms_total / 1e3) / 1e9
    # dominant kernel: the sweep (one launch per step on 1 GPU and with the
    # fused halo, its peer stores included; with NCCL the sum of the step's
    # three range launches, the overlapped halo excluded)
    if sweep_only:
        sweep_ms = sum(a.elapsed_time(b) for a, b in sweep_only) / len(sweep_only)
    else:  # the step's boundary + interior sweep launches, halo excluded
        sweep_ms = sum(sum(a.elapsed_time(b) for a, b in st) for st in multi_sweeps) / len(multi_sweeps)
    local_cells = p.dims.interior_cells
    achieved = BYTES_PER_UPDATE * local_cells / (sweep_ms / 1e3) / 1e9
    halo_stall = None
    if world > 1:
        # this rank's average stall per step waiting for its neighbours'
        # planes (fused: the flag wait; NCCL: the exchange + unpack), then
        # every rank's value gathered: overlap shows as a small fraction of
        # the step
        mine = sum(a.elapsed_time(b) for a, b in halo_waits) / max(1, len(halo_waits))
        allw = torch.zeros(world, dtype=torch.float64, device=dev)
        allw[rank] = mine
        dist.all_reduce(allw)
        per = [float(v) for v in allw.cpu()]
        halo_stall = {"ms_per_step_by_rank": per, "max": max(per), "mean": sum(per) / world,
                      "frac_of_step": max(per) / (ms_total / args.steps),
                      "what": "flag wait kernel (fused peer halo)" if halo is not None else
                              "stream wait on the NCCL exchange + unpack"}
    peak, peak_src = _peaks()
    roofline = {
        "bound": "hbm",
        "achieved": achieved,
        "peak": peak,
        "unit": "GB/s",
        "frac": achieved / peak,
        "traffic": _traffic(f"line_jacobi_{nx}x{ny}x{p.dims.nz}"),
        "traffic_source": "profiles/ncu_traffic.json: dram__bytes_read.sum + dram__bytes_write.sum of one launch "
                          "from the committed ncu --set full capture of this shape (null when none)",
        "kernel": f"psm::line_jacobi_zmarch_kernel<{nx},1,{2 if halo is not None else 0}> (line Jacobi sweep, fused "
                  "residual norm + x ghosts" + (", peer-halo stores)" if halo is not None else ")"),
        "bytes_per_launch": BYTES_PER_UPDATE * local_cells,
        "avg_launch_ms": sweep_ms,
        "peak_source": peak_src,
        "frac_of_nominal_8000": achieved / 8000.0,
    }
    clocks = clk.summary()

    # ---- e2e through the public API with host buffers ---------------------
    e2e = None
    if not args.no_e2e:
        e2e = _e2e(args, dom, cfg, cache, dev, world, rank)

    # ---- the north-star grid: 512^3 line-Jacobi sweep, device-timed --------
    north = None
    if world == 1 and not args.no_north_star:
        del dom, p, plan, dp
        torch.cuda.empty_cache()
        north = _north_star(args, dev)

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        port = CpuPort(nx, ny, 8)
        v, n, el = port.rate(seconds=args.cpu_seconds)
        cpu = port.describe(v, n, el)
        cpu["reference_py"] = _reference_py(nx)

    if rank == 0:
        line = {
            "metric": METRIC,
            "value": value,
            "unit": UNIT,
            "n_gpus": world,
            "steps": args.steps,
            "warmup": args.warmup,
            "ms_per_step": ms_total / args.steps,
            "higher_is_better": True,
            "scaling": "strong",
            "vs_baseline": None,
            "dtype": "f64",
            "data": "synthetic: u0 ~ U[0,1), f ~ N(0,1) from a per-rank seeded device generator",
            "config": {
                "workload": f"C5: {nx}x{ny}x{nz} uniform grid, line block Jacobi, z-slabs over {world} GPU(s)",
                "global_shape": [nx, ny, nz],
                "block_dims": [nx, 1, 1],
                "omega": 0.8,
                "parallelism": f"z-slab x{world}",
                "step": "sweep (+fused norm, x ghosts) + swap + physical ghosts" + (
                    "" if world == 1 else
                    " + halo fused into the sweep (peer-memory stores, step flags)" if halo is not None else
                    " + NCCL halo, overlapped"),
                "halo": None if world == 1 else halo_mode,
                "l2": f"no flush: inputs {BYTES_PER_UPDATE * local_cells / 1e9:.1f} GB per sweep per GPU "
                      ">> 126 MB L2",
            },
            "roofline": roofline,
            "north_star_512": north,
            "halo_stall": halo_stall,
            "cpu_baseline": cpu,
            "e2e": e2e,
            "gpu_launches": int(launches),
            "clocks": clocks,
        }
        print(json.dumps(line), flush=True)


def _north_star(args, dev, n=512, sweeps=20):
    """The north-star target (BASELINE.json): one 512^3 line-Jacobi sweep on
    one B200, >= 70% of the 8 TB/s HBM roofline.  Timed like the headline:
    CUDA events around each sweep launch on the launching stream, after
    warm-up; inputs (3.2 GB per sweep) far exceed L2."""
    import torch

    import paper_1208_1975_b200 as ps
    from paper_1208_1975_b200 import _lib
    from paper_1208_1975_b200.dist import SlabDomain
    from paper_1208_1975_b200.smoother import _Plan

    dom = SlabDomain((n, n, n), 0, 1, device=dev)
    p = dom.patch
    gen = torch.Generator(device=dev)
    gen.manual_seed(512)
    p.interior.copy_(torch.rand(p.interior.shape, generator=gen, device=dev, dtype=torch.float64))
    p.f.copy_(torch.randn(p.f.shape, generator=gen, device=dev, dtype=torch.float64))
    cfg = ps.SmootherConfig(scheme="block_jacobi", block_dims=(n, 1, 1), omega=0.8, steps=1,
                            strategy=ps.ExecutionStrategy.device())
    dp = _Plan(dom.level, cfg, ps.InverseCache()).dev
    dp.reserve(2)
    lib = _lib.load()
    stream = torch.cuda.current_stream(dev)
    act = (ctypes.c_ubyte * 1)()
    dp.refresh(_lib.GHOST_ALL)
    pairs = []
    for s in range(args.warmup + sweeps):
        act[0] = p._active
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        _lib.check(lib.psm_jacobi_sweep(dp.handle, act, 0.8, s % 2, ctypes.c_void_p(stream.cuda_stream)),
                   "jacobi_sweep")
        e1.record(stream)
        if s >= args.warmup:
            pairs.append((e0, e1))
        p.swap_buffers()
        dp.refresh(_lib.GHOST_ALL | _lib.GHOST_SKIP_X)
    torch.cuda.synchronize(dev)
    ms = sorted(a.elapsed_time(b) for a, b in pairs)
    avg = sum(ms) / len(ms)
    cells = n ** 3
    gbs = BYTES_PER_UPDATE * cells / (avg / 1e3) / 1e9
    peak, src = _peaks()
    out = {
        "workload": f"{n}^3 single patch, line block Jacobi (block_dims ({n},1,1), omega 0.8), 1 GPU",
        "kernel": f"psm::line_jacobi_zmarch_kernel<{n},1,0>",
        "sweeps": sweeps,
        "avg_sweep_ms": avg,
        "median_sweep_ms": ms[len(ms) // 2],
        "Gupdates_per_s": cells / (avg / 1e3) / 1e9,
        "achieved_GBps": gbs,
        "frac_of_nominal_8000": gbs / 8000.0,
        "frac_of_measured": gbs / peak,
        "peak_source": src,
        "target": ">= 0.70 of 8 TB/s",
    }
    del dom, p, dp
    torch.cuda.empty_cache()
    return out


def _reference_py(nx, ny=16, nz=8, repeat=2):
    """The reference smoother itself (patchsmooth, pure Python/numpy, from
    baseline/_ref, installed by __graft_entry__.build()) on a bounded slab of
    the workload, through its own harness: build_level, seed_initial_guess,
    run_bench (warm inverse cache, min of `repeat` smooth() calls incl.
    ghosts and history), serial strategy (its fastest: SURVEY F7)."""
    ref = os.path.join(ROOT, "baseline", "_ref")
    if not os.path.isdir(os.path.join(ref, "patchsmooth")):
        return {"unavailable": "baseline/_ref/patchsmooth not installed (run __graft_entry__.build() where "
                               "/root/reference exists)"}
    sys.path.insert(0, ref)
    try:
        import patchsmooth as R
    finally:
        sys.path.remove(ref)
    level = R.build_level([(nx, ny, nz)])
    R.seed_initial_guess(level, 42)
    cfg = R.SmootherConfig(scheme="block_jacobi", block_dims=(nx, 1, 1), steps=1)
    t0 = time.perf_counter()
    rec = R.run_bench(level, [cfg], repeat=repeat, label=f"{nx}x{ny}x{nz}")[0]
    total = time.perf_counter() - t0
    return {
        "value": rec.cells_per_second / 1e9,
        "unit": UNIT,
        "cores": 1,
        "kind": "reference",
        "sample": f"patchsmooth {getattr(R, '__version__', '?')} run_bench: min of {repeat} smooth() calls "
                  f"(1 line-Jacobi step + ghosts + 2 history norms) on a {nx}x{ny}x{nz} slab, serial strategy, "
                  f"inverse cache warmed outside the timing ({total:.1f} s in all)",
        "wall_seconds": rec.wall_seconds,
        "host_cpus": os.cpu_count(),
    }


def _e2e(args, dom, cfg, cache, dev, world, rank):
    import torch
    import torch.distributed as dist

    import paper_1208_1975_b200 as ps
    from paper_1208_1975_b200.dist import dist_smooth

    p = dom.patch
    sweeps = args.e2e_sweeps
    ecfg = ps.SmootherConfig(scheme="block_jacobi", block_dims=cfg.block_dims, omega=0.8, steps=sweeps,
                             strategy=cfg.strategy)
    host_u = torch.empty(p._bufs[0].shape, dtype=torch.float64, pin_memory=True)
    host_f = torch.empty(p._f.shape, dtype=torch.float64, pin_memory=True)
    host_u.copy_(p._bufs[p._active])
    host_f.copy_(p._f)
    out_u = torch.empty_like(host_u, pin_memory=True)

    def call():
        p._active = 0
        p._bufs[0].copy_(host_u, non_blocking=True)
        p._f.copy_(host_f, non_blocking=True)
        hist = dist_smooth(dom, ecfg, cache) if world > 1 else ps.smooth(dom.level, ecfg, cache)[1]
        out_u.copy_(p._bufs[p._active], non_blocking=True)
        torch.cuda.current_stream(dev).synchronize()
        return hist

    call()
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize(dev)
    t0 = time.perf_counter()
    for _ in range(args.e2e_calls):
        hist = call()
    el = time.perf_counter() - t0
    t = torch.tensor([el], dtype=torch.float64, device=dev)
    if world > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    el = float(t.item())
    nx, ny, nz = dom.global_shape
    value = nx * ny * nz * sweeps * args.e2e_calls / el / 1e9
    h2d = (host_u.numel() + host_f.numel()) * 8 * world
    d2h = (out_u.numel() * 8 + (sweeps + 1) * 8) * world
    assert all(math.isfinite(h) for h in hist)
    return {
        "value": value,
        "unit": UNIT,
        "h2d_bytes_per_step": h2d,
        "d2h_bytes_per_step": d2h,
        "step": f"one smooth() call: H2D u,f (pinned) + {sweeps} sweeps with history + D2H u + history",
        "calls": args.e2e_calls,
        "seconds": el,
    }


def main():
    args = parse()
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local_rank = int(os.environ.get("LOCAL_RANK", "0"))
    if world != args.gpus and world > 1:
        print(f"warning: WORLD_SIZE={world} but --gpus={args.gpus}", file=sys.stderr)
    if args.impl == "reference":
        run_reference(args, rank, world)
        return
    if world > 1:
        import torch
        import torch.distributed as dist

        # PSM_DIST_BACKEND=gloo runs several ranks on fewer GPUs (halo staged
        # through host memory) to exercise the multi-rank path on one GPU
        backend = os.environ.get("PSM_DIST_BACKEND", "nccl")
        local_rank = local_rank % max(1, torch.cuda.device_count())
        torch.cuda.set_device(local_rank)
        if backend == "nccl":
            dist.init_process_group("nccl", device_id=torch.device("cuda", local_rank))
        else:
            dist.init_process_group(backend)
    try:
        run_ours(args, rank, world, local_rank)
    finally:
        if world > 1:
            import torch.distributed as dist

            dist.destroy_process_group()


if __name__ == "__main__":
    main()
