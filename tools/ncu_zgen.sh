#!/bin/bash
export PATCHSMOOTH_MAX_CELLS=${PATCHSMOOTH_MAX_CELLS:-100000000000}  # device-sized levels
# full ncu capture of one runtime-nx line-Jacobi sweep (zgen) on the mixed
# Table-2 patch set: tools/ncu_zgen.sh OUT
OUT=${1:-prof_zgen}
mkdir -p gpurun_out
cat > /tmp/zgen_one.py <<PY
import sys; sys.path.insert(0, '.')
import torch, paper_1208_1975_b200 as ps
from paper_1208_1975_b200.smoother import _Plan, _run
lv = ps.build_patch_set(ps.PatchSetSpec.mixed_table2())
for p in lv.patches:
    p.interior.copy_(torch.rand(p.interior.shape, dtype=torch.float64, device="cuda"))
    p.f.copy_(torch.randn(p.f.shape, dtype=torch.float64, device="cuda"))
cfg = ps.SmootherConfig(scheme="block_jacobi", block_dims=(96, 1, 1))
plan = _Plan(lv, cfg, ps.InverseCache())
_run(lv, cfg, plan, 3, False, {})
torch.cuda.synchronize()
PY
timeout -s KILL 600 ncu --set full --clock-control none --import-source on -k regex:zgen -s 1 -c 1 -o gpurun_out/$OUT python /tmp/zgen_one.py > gpurun_out/$OUT.log 2>&1
echo "ncu rc=$?"
python tools/ncu_summary.py gpurun_out/$OUT.ncu-rep > gpurun_out/${OUT}_summary.txt 2>&1
python tools/ncu_src_top.py gpurun_out/$OUT.ncu-rep 30 >> gpurun_out/${OUT}_summary.txt 2>&1
