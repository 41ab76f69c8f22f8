"""Per-configuration device timing of every BASELINE.json config on one GPU.

One "step" is what the reference's smoother step does (smoother.py:138-169):
the sweep plus the ghost refresh, without history.  Timed with CUDA events on
the current stream over K steps in graph replay (the steady state of repeated
smooth() calls) after W warm-up steps; prints one JSON line
per (config, scheme) with updates/s, GB/s at the 24 B/update algorithmic
traffic, and for plane blocks the algorithmic fp64 TFLOP/s.

    python tools/bench_configs.py [--only C3] [--steps K] [--warmup W]
"""
from __future__ import annotations

import argparse
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

os.environ.setdefault("PATCHSMOOTH_MAX_CELLS", str(10**11))  # device-sized levels
import torch  # noqa: E402

import paper_1208_1975_b200 as ps  # noqa: E402
from paper_1208_1975_b200.smoother import _Plan, _run  # noqa: E402
from paper_1208_1975_b200.workloads import build_lattice  # noqa: E402


def _fill(level, seed=0):
    g = torch.Generator(device="cuda")
    g.manual_seed(seed)
    for p in level.patches:
        p.interior.copy_(torch.rand(p.interior.shape, dtype=torch.float64, device="cuda", generator=g))
        p.f.copy_(torch.randn(p.f.shape, dtype=torch.float64, device="cuda", generator=g))


def plane_flops(nx):
    # two DST transforms (2*nx each) + modal Thomas (5) + residual (8) + relax (2)
    return 4 * nx + 15


def time_steps(level, cfg, steps, warmup):
    """Device time per step of a `steps`-step sequence in its steady state:
    the first call with a new step count runs eagerly, the second captures
    the CUDA graph, the timed third call replays it (as repeated smooth()
    calls do)."""
    plan = _Plan(level, cfg, ps.InverseCache())
    ps.smoother._run(level, cfg, plan, warmup, False, None)
    for _ in range(2):
        _run(level, cfg, plan, steps, False, None)
    torch.cuda.synchronize()
    s = torch.cuda.current_stream()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(s)
    _run(level, cfg, plan, steps, False, None)
    e1.record(s)
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / steps, plan


def time_smooth(level, cfg, reps=20):
    """Full smooth() calls (history included, one D2H each), device-timed,
    with one warm InverseCache like the reference's run_bench (bench.py:211):
    the first call runs eagerly, the second captures the CUDA graph."""
    cache = ps.InverseCache()
    for _ in range(3):
        ps.smooth(level, cfg, cache)
    torch.cuda.synchronize()
    s = torch.cuda.current_stream()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(s)
    for _ in range(reps):
        ps.smooth(level, cfg, cache)
    e1.record(s)
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps


CONFIGS = {
    "C1": dict(desc="64^3 single patch, line block Jacobi, 10 sweeps (smooth() incl. history)",
               build=lambda: ps.build_level([(64, 64, 64)]), runs=[("block_jacobi", "line", None)], smooth_steps=10),
    "C2": dict(desc="256^3 single patch, line GS: chaotic vs colour(wavefront)-ordered",
               build=lambda: ps.build_level([(256, 256, 256)]),
               runs=[("chaotic_block_gs", "line", "chaotic"), ("chaotic_block_gs", "line", "wavefront")]),
    "C3": dict(desc="512^3 single patch, plane block Jacobi, exact plane inverse",
               build=lambda: ps.build_level([(512, 512, 512)]),
               runs=[("block_jacobi", "plane", None), ("block_jacobi", "plane", "dst")]),
    "C4": dict(desc="AMR-style 4x4x4 lattice of 128^3 patches (288 interface copies), line/plane GS",
               build=lambda: build_lattice((4, 4, 4), (128, 128, 128)),
               runs=[("chaotic_block_gs", "line", "wavefront"), ("chaotic_block_gs", "line", "chaotic"),
                     ("chaotic_block_gs", "plane", "wavefront"), ("block_jacobi", "line", None)]),
    "F1": dict(desc="SURVEY f1: 512^3 single patch, box (cubic) blocks of the paper's Algorithm 2",
               build=lambda: ps.build_level([(512, 512, 512)]),
               runs=[("block_jacobi", (8, 8, 8), None), ("block_jacobi", (4, 4, 4), None),
                     ("block_jacobi", (2, 2, 2), None), ("chaotic_block_gs", (8, 8, 8), "wavefront")]),
    "F3": dict(desc="SURVEY f3 / paper Table 2: mixed set, 16 patches each of 64^3..96^3 abutting along x",
               build=lambda: ps.build_patch_set(ps.PatchSetSpec.mixed_table2()),
               runs=[("block_jacobi", (96, 1, 1), None), ("chaotic_block_gs", (96, 1, 1), "wavefront"),
                     ("chaotic_block_gs", (96, 1, 1), "chaotic"), ("block_jacobi", (96, 96, 1), None),
                     ("block_jacobi", (8, 8, 8), None)]),
    "C5": dict(desc="1024^3 uniform grid, line Jacobi, 1 GPU",
               build=lambda: ps.build_level([(1024, 1024, 1024)]), runs=[("block_jacobi", "line", None)]),
}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--only", default=None)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--runs", default=None, help="comma list of run indices within each config")
    a = ap.parse_args()
    names = a.only.split(",") if a.only else list(CONFIGS)
    for name in names:
        C = CONFIGS[name]
        level = C["build"]()
        _fill(level)
        cells = level.interior_cells
        p0 = level.patches[0].dims
        sel = [int(x) for x in a.runs.split(",")] if a.runs else range(len(C["runs"]))
        for ri, (scheme, kind, mode) in enumerate(C["runs"]):
            if ri not in sel:
                continue
            if isinstance(kind, tuple):  # explicit block dims
                bd = kind
                kind = ("line" if kind[1:] == (1, 1) else "plane" if kind[2] == 1 else
                        "box" + "x".join(str(b) for b in kind))
            else:
                bd = (p0.nx, 1, 1) if kind == "line" else (p0.nx, p0.ny, 1)
            solver = "dst" if mode == "dst" else "auto"
            gs_mode = mode if mode in ("wavefront", "chaotic") else "wavefront"
            strat = ps.ExecutionStrategy.device(gs_mode=gs_mode)
            cfg = ps.SmootherConfig(scheme=scheme, block_dims=bd, strategy=strat)
            prev = ps.plane_solver(solver)
            try:
                ms, plan = time_steps(level, cfg, a.steps, a.warmup)
            finally:
                ps.plane_solver(prev)
            rec = {"config": name, "desc": C["desc"], "scheme": scheme, "block": kind, "gs_mode": mode,
                   "cells": cells, "ms_per_step": round(ms, 4), "Gupdates_per_s": round(cells / ms / 1e6, 2),
                   "GBps_at_24B": round(24 * cells / ms / 1e6, 1)}
            if kind == "plane":
                rec["plane_solver"] = solver
                if solver == "dst":
                    rec["TFLOPs_alg"] = round(plane_flops(p0.nx) * cells / ms / 1e9, 2)
            if C.get("smooth_steps"):
                cfg2 = ps.SmootherConfig(scheme=scheme, block_dims=bd, strategy=strat, steps=C["smooth_steps"])
                tms = time_smooth(level, cfg2)
                rec["smooth_call_ms"] = round(tms, 4)
                rec["smooth_Gupdates_per_s"] = round(cells * C["smooth_steps"] / tms / 1e6, 2)
            print(json.dumps(rec), flush=True)
            del plan
        del level
        torch.cuda.empty_cache()


if __name__ == "__main__":
    main()
