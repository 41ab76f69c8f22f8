"""Phase timings of the one-tile-per-CTA line-Jacobi kernel on a 64^3 level.

Build the instrumented variant (globaltimer stamps, printf from CTAs 0 and
77 per tile: phase A = loads + residual, B = segment solves, C = relax and
stores) and point the binding at it:

  nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -Xcompiler -fPIC \
       -DPSM_NX_TIMING -c -o build/variant/psm_line_t.o paper_1208_1975_b200/csrc/psm_line.cu
  nvcc -gencode arch=compute_100a,code=sm_100a -shared -o build/variant/libpsmooth_t.so \
       $(ls build/obj/*.o | grep -v psm_line.o) build/variant/psm_line_t.o -lcudart
  PSM_LIB=$PWD/build/variant/libpsmooth_t.so python tools/nx_timing_probe.py
"""
import sys

import torch

sys.path.insert(0, ".")
import paper_1208_1975_b200 as ps  # noqa: E402
from paper_1208_1975_b200.smoother import _Plan, _run  # noqa: E402

lv = ps.build_level([(64, 64, 64)])
ps.seed_initial_guess(lv, seed=1)
cfg = ps.SmootherConfig(scheme="block_jacobi", block_dims=(64, 1, 1), steps=3)
plan = _Plan(lv, cfg, ps.InverseCache())
for i in range(3):
    _run(lv, cfg, plan, 3, False, None)
    torch.cuda.synchronize()
    print("---- call", i, flush=True)
