#!/bin/bash
# ncu --set full of the C4 plane-GS kernels, one capture each: tools/ncu_plane_gs.sh PREFIX
export PATCHSMOOTH_MAX_CELLS=${PATCHSMOOTH_MAX_CELLS:-100000000000}
PRE=${1:-prof_pgs}
mkdir -p gpurun_out
for spec in "fwd:dst_tile_kernel:0" "bwd:dst_tile_kernel:1" "chain:plane_gs_chain:0"; do
  IFS=: read name pat skip <<< "$spec"
  timeout -s KILL 600 ncu --set full --import-source on --clock-control none -k "regex:${pat}" --launch-skip $skip -c 1 \
    -o gpurun_out/${PRE}_$name -f python tools/bench_configs.py --only C4 --runs 2 --steps 1 --warmup 1 \
    > gpurun_out/${PRE}_$name.log 2>&1
  echo "== $name rc=$?"
  python tools/ncu_summary.py gpurun_out/${PRE}_$name.ncu-rep 2>&1 | head -45
done
