"""Latency probe of the pipelined line GS: sweep time vs plane count, to
separate per-row cost (nz=1), intra-CTA hand-off (nz<=8) and cross-CTA
hand-off (nz>8).  python tools/gs_probe.py"""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
os.environ.setdefault("PATCHSMOOTH_MAX_CELLS", str(10**11))  # device-sized levels
import torch  # noqa: E402

import paper_1208_1975_b200 as ps  # noqa: E402
from paper_1208_1975_b200.smoother import _Plan  # noqa: E402


def sweep_ms(shape, mode="wavefront", reps=20):
    lv = ps.build_level([shape])
    p = lv.patches[0]
    p.interior.copy_(torch.rand(p.interior.shape, dtype=torch.float64, device="cuda"))
    p.f.copy_(torch.randn(p.f.shape, dtype=torch.float64, device="cuda"))
    cfg = ps.SmootherConfig(scheme="chaotic_block_gs", block_dims=(shape[0], 1, 1),
                            strategy=ps.ExecutionStrategy.device(gs_mode=mode))
    plan = _Plan(lv, cfg, ps.InverseCache())
    from paper_1208_1975_b200 import _lib
    m = _lib.GS_CHAOTIC if mode == "chaotic" else _lib.GS_WAVEFRONT
    for _ in range(3):
        plan.dev.gs(1.0, m)
    torch.cuda.synchronize()
    s = torch.cuda.current_stream()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(s)
    for _ in range(reps):
        plan.dev.gs(1.0, m)
    e1.record(s)
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps


if __name__ == "__main__":
    for nx in (256, 128):
        for nz in (1, 2, 8, 16, 64, nx):
            ms = sweep_ms((nx, nx, nz))
            print(json.dumps({"shape": [nx, nx, nz], "ms": round(ms, 4),
                              "us_per_wavefront_step": round(1e3 * ms / (nx + nz - 1), 3)}), flush=True)
