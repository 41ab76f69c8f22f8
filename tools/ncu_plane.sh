#!/bin/bash
export PATCHSMOOTH_MAX_CELLS=${PATCHSMOOTH_MAX_CELLS:-100000000000}  # device-sized levels
# ncu of the plane-Jacobi kernels at NX^3 (launch list + one full capture of the banded solve)
NX=${1:-512}; OUT=${2:-prof_plane}
mkdir -p gpurun_out
cat > /tmp/plane_one.py <<PY
import sys; sys.path.insert(0, '.')
import torch, paper_1208_1975_b200 as ps
from paper_1208_1975_b200.smoother import _Plan, _run
lv = ps.build_level([($NX, $NX, $NX)])
p = lv.patches[0]
p.interior.copy_(torch.rand(p.interior.shape, dtype=torch.float64, device="cuda"))
p.f.copy_(torch.randn(p.f.shape, dtype=torch.float64, device="cuda"))
cfg = ps.SmootherConfig(scheme="block_jacobi", block_dims=($NX, $NX, 1))
plan = _Plan(lv, cfg, ps.InverseCache())
_run(lv, cfg, plan, 3, False, None)
torch.cuda.synchronize()
PY
timeout -s KILL 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/${OUT}_launches.csv python /tmp/plane_one.py > /dev/null 2>&1
timeout -s KILL 600 ncu --set full --clock-control none --import-source on -k regex:plane_band -s 1 -c 1 -o gpurun_out/$OUT python /tmp/plane_one.py > gpurun_out/$OUT.log 2>&1
echo "ncu rc=$?"
