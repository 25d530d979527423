#!/bin/bash
# compute-sanitizer over the hot path's kernels (tools/sanitize_cases.py):
# memcheck, initcheck, synccheck and racecheck, one log per tool and case
# under gpurun_out/sanitize/ (summaries copied to profiles/ by hand).
# PAPER:122 (Sec. 3) names thread contention as the hazard of the method's
# parallelisation; racecheck covers the shared-memory ring, synccheck the
# barriers, memcheck / initcheck the TMA boxes and the partial records.
#   bash tools/sanitize.sh [case ...]
cd "$(dirname "$0")/.."
OUT=gpurun_out/sanitize
mkdir -p $OUT
CASES=${*:-c1 3d 2d v2 pipe modes slab}
CS=/usr/local/cuda/bin/compute-sanitizer
TOOLS=${TOOLS:-memcheck initcheck synccheck racecheck}
for tool in $TOOLS; do
  for c in $CASES; do
    extra=""
    [ $tool = memcheck ] && extra="--leak-check no"
    [ $tool = racecheck ] && extra="--racecheck-report all"
    timeout 900 $CS --tool $tool $extra --error-exitcode 9 --print-limit 20 \
      python tools/sanitize_cases.py $c > $OUT/${tool}_${c}.log 2>&1
    rc=$?
    summ=$(grep -E "ERROR SUMMARY|RACECHECK SUMMARY|hazard" $OUT/${tool}_${c}.log | tail -1)
    echo "$tool $c rc=$rc $summ" | tee -a $OUT/summary.txt
  done
done
