#!/bin/bash
export PATCHSMOOTH_MAX_CELLS=${PATCHSMOOTH_MAX_CELLS:-100000000000}  # device-sized levels
# compute-sanitizer memcheck / racecheck / synccheck / initcheck over small
# deterministic invocations of every kernel family (tools/sanitize_cases.py).
# The chaotic GS schedule is racy by design: it runs under
# memcheck and synccheck only.  Output: gpurun_out/sanitizer.log
mkdir -p gpurun_out
LOG=gpurun_out/sanitizer.log
: > $LOG
CS=/usr/local/cuda/bin/compute-sanitizer
run() {
  tool=$1; shift
  echo "=== $tool $* $EXTRA" | tee -a $LOG
  timeout 1200 $CS --tool $tool --error-exitcode 99 "$@" python tools/sanitize_cases.py $EXTRA >> $LOG 2>&1
  rc=$?
  echo "=== $tool $EXTRA rc=$rc" | tee -a $LOG
}
EXTRA="--chaotic" run memcheck --leak-check no
# racecheck one case at a time, so each kernel family gets its own summary
for c in zmarch_line_jacobi zmarch_line_jacobi_256 zgen_line_jacobi odd_line_jacobi gs_pipe_wavefront gs_pipe_odd_nx \
         plane_band_jacobi plane_gs plane_gs_mixed box_jacobi box_gs ghosts_lattice_jacobi gs_multisweep \
         plane_gs_dst_chain plane_jacobi_dst box_gs_persistent api_primitives box_jacobi_4 box_jacobi_odd; do
  EXTRA="--only $c" run racecheck --racecheck-report hazard --print-limit 4
done
EXTRA="--chaotic" run synccheck
EXTRA="" run initcheck
grep -E "ERROR SUMMARY|RACECHECK SUMMARY|=== " $LOG
