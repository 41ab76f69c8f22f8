#!/bin/bash
export PATCHSMOOTH_MAX_CELLS=${PATCHSMOOTH_MAX_CELLS:-100000000000}  # device-sized levels
# full ncu capture of one box-block sweep: tools/ncu_box.sh N B OUT [SCHEME]
N=${1:-256}; B=${2:-8}; OUT=${3:-prof_box}; SCHEME=${4:-block_jacobi}
mkdir -p gpurun_out
cat > /tmp/box_one.py <<PY
import sys; sys.path.insert(0, '.')
import torch, paper_1208_1975_b200 as ps
from paper_1208_1975_b200.smoother import _Plan, _run
lv = ps.build_level([($N, $N, $N)])
p = lv.patches[0]
p.interior.copy_(torch.rand(p.interior.shape, dtype=torch.float64, device="cuda"))
p.f.copy_(torch.randn(p.f.shape, dtype=torch.float64, device="cuda"))
cfg = ps.SmootherConfig(scheme="$SCHEME", block_dims=($B, $B, $B))
plan = _Plan(lv, cfg, ps.InverseCache())
_run(lv, cfg, plan, 3, False, {})
torch.cuda.synchronize()
PY
timeout -s KILL 600 ncu --set full --clock-control none --import-source on -k regex:box_sweep -s 1 -c 1 -o gpurun_out/$OUT python /tmp/box_one.py > gpurun_out/$OUT.log 2>&1
echo "ncu rc=$?"
python tools/ncu_summary.py gpurun_out/$OUT.ncu-rep > gpurun_out/${OUT}_summary.txt 2>&1
python tools/ncu_src_top.py gpurun_out/$OUT.ncu-rep 25 >> gpurun_out/${OUT}_summary.txt 2>&1
