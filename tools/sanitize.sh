#!/bin/bash
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
  echo "=== $tool $*" | tee -a $LOG
  timeout 1200 $CS --tool $tool --error-exitcode 99 "$@" python tools/sanitize_cases.py $EXTRA >> $LOG 2>&1
  rc=$?
  echo "=== $tool rc=$rc" | tee -a $LOG
}
EXTRA="--chaotic" run memcheck --leak-check no
EXTRA="" run racecheck --racecheck-report all
EXTRA="--chaotic" run synccheck
EXTRA="" run initcheck
grep -E "ERROR SUMMARY|RACECHECK SUMMARY|=== " $LOG
