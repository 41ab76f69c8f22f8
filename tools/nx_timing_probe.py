"""Phase timings of the one-tile-per-CTA line-Jacobi kernel on a 64^3 level.

Build the instrumented variant (globaltimer stamps, one printf per tile:
absolute start/end, phase A = loads + residual, B = segment solves, C =
relax and stores) and point the binding at it:

  nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -Xcompiler -fPIC \\
       -DPSM_NX_TIMING -c -o build/variant/psm_line_t.o paper_1208_1975_b200/csrc/psm_line.cu
  nvcc -gencode arch=compute_100a,code=sm_100a -shared -o build/variant/libpsmooth_t.so \\
       $(ls build/obj/*.o | grep -v psm_line.o) build/variant/psm_line_t.o -lcudart
  PSM_LIB=$PWD/build/variant/libpsmooth_t.so python tools/nx_timing_probe.py

Prints, per launch, the CTA start/end spread and the median phase times.
"""
import os
import re
import subprocess
import sys

if os.environ.get("_NX_CHILD") != "1":
    env = dict(os.environ, _NX_CHILD="1")
    out = subprocess.run([sys.executable, __file__], env=env, capture_output=True, text=True).stdout
    launches, cur = [], []
    for line in out.splitlines():
        m = re.search(r"start (\d+) end (\d+)  A (\d+)  B (\d+)  C (\d+)", line)
        if m:
            cur.append(tuple(int(x) for x in m.groups()))
        elif line.startswith("---- launch"):
            launches.append(cur)
            cur = []
    for i, L in enumerate(launches):
        if not L:
            continue
        s0 = min(x[0] for x in L)
        med = lambda k: sorted(x[k] for x in L)[len(L) // 2]  # noqa: E731
        print(f"launch {i}: {len(L)} tiles, CTA starts spread {max(x[0] for x in L) - s0} ns, "
              f"last end {max(x[1] for x in L) - s0} ns after first start; median A {med(2)} B {med(3)} C {med(4)} ns")
    sys.exit(0)

import torch  # noqa: E402

sys.path.insert(0, ".")
import paper_1208_1975_b200 as ps  # noqa: E402
from paper_1208_1975_b200.smoother import _Plan, _run  # noqa: E402

lv = ps.build_level([(64, 64, 64)])
ps.seed_initial_guess(lv, seed=1)
cfg = ps.SmootherConfig(scheme="block_jacobi", block_dims=(64, 1, 1), steps=1)
plan = _Plan(lv, cfg, ps.InverseCache())
for i in range(4):
    _run(lv, cfg, plan, 1, False, None)
    torch.cuda.synchronize()
    print("---- launch", i, flush=True)
