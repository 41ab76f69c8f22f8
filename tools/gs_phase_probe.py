"""Phase timing of the pipelined line GS row loop (block 0, warp 0, lane 0),
from a profiling build: tools/build_prof.sh; then
PSM_LIB=paper_1208_1975_b200/libpsmooth_prof.so python tools/gs_phase_probe.py"""
import ctypes, json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from tools.gs_probe import sweep_ms  # noqa: E402
from paper_1208_1975_b200 import _lib  # noqa: E402

names = ["loop", "issue", "cp_wait", "loads+zm", "residual", "thomas", "pcr", "x+relax", "handoff+store"]
lib = _lib.load()
buf = (ctypes.c_longlong * 16)()
for shape in [(256, 256, 1), (256, 256, 8), (128, 128, 1), (128, 128, 7), (256, 256, 256)]:
    lib.psm_debug_gs_profile(buf, 1)
    ms = sweep_ms(shape, reps=1)
    lib.psm_debug_gs_profile(buf, 1)
    sweeps = 4  # 3 warm-up + 1 timed in sweep_ms(reps=1)
    rows = shape[1] * sweeps
    print(json.dumps({"shape": shape, "ms": round(ms, 4),
                      "cycles_per_row": {n: round(buf[i] / rows, 1) for i, n in enumerate(names)},
                      "total": round(sum(buf[i] for i in range(1, 9)) / rows, 1)}))
