"""Kernel-level timing of the line-Jacobi sweep (CUDA events, no ghosts)."""
import ctypes, sys, os, json
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_1208_1975_b200 as ps
from paper_1208_1975_b200 import _lib
from paper_1208_1975_b200.smoother import _Plan

def run(shape, reps=10, faces=None):
    nx, ny, nz = shape
    lv = ps.Level([ps.Patch(ps.PatchDims(*shape))])
    p = lv.patches[0]
    p.interior.copy_(torch.rand(p.interior.shape, dtype=torch.float64, device="cuda"))
    p.f.copy_(torch.randn(p.f.shape, dtype=torch.float64, device="cuda"))
    st = ps.Stencil7() if faces is None else ps.Stencil7(6.0, faces)
    cfg = ps.SmootherConfig(scheme="block_jacobi", block_dims=(nx, 1, 1), stencil=st)
    plan = _Plan(lv, cfg, ps.InverseCache())
    dp = plan.dev; dp.reserve(1); dp.refresh()
    lib = _lib.load()
    act = (ctypes.c_ubyte * 1)(0)
    s = torch.cuda.current_stream()
    for _ in range(3):
        _lib.check(lib.psm_jacobi_sweep(dp.handle, act, 0.8, 0, ctypes.c_void_p(s.cuda_stream)))
    torch.cuda.synchronize()
    e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
    e0.record(s)
    for _ in range(reps):
        lib.psm_jacobi_sweep(dp.handle, act, 0.8, 0, ctypes.c_void_p(s.cuda_stream))
    e1.record(s); torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / reps
    cells = nx * ny * nz
    print(json.dumps({"shape": shape, "unit_faces": faces is None, "ms": round(ms, 4), "GBps": round(24 * cells / ms / 1e6, 1),
                      "Gupd": round(cells / ms / 1e6, 2)}), flush=True)
    del plan, dp, lv, p
    torch.cuda.empty_cache()

if __name__ == "__main__":
    for sh in [(1024, 1024, 1024), (512, 512, 512), (256, 256, 256), (128, 128, 128), (64, 64, 64), (1024, 1024, 64)]:
        run(sh)
    run((512, 512, 512), faces=(-1.0, -1.0, -1.0, -1.0, -1.0, -0.9999))
