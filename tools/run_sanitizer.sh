#!/bin/bash
# compute-sanitizer racecheck / synccheck / memcheck over tools/sanitize_cases.py
# (one small invocation per kernel); logs -> gpurun_out/sanitizer/<tool>_<case>.log
out=gpurun_out/sanitizer
mkdir -p $out
export SOM_SPIN_TIMEOUT_MS=900000
CASES=${CASES:-"k1 k2 k3 k4 k5 k6 k10 map_exact map_sparse map_tc metrics batch"}
TOOLS=${TOOLS:-"memcheck racecheck synccheck"}
for tool in $TOOLS; do
  for c in $CASES; do
    extra=""
    [ "$tool" = "memcheck" ] && extra="--leak-check no"
    [ "$tool" = "racecheck" ] && extra="--racecheck-report all"
    start=$(date +%s)
    timeout ${CASE_TIMEOUT:-420} compute-sanitizer --tool $tool $extra --error-exitcode 9 \
        python tools/sanitize_cases.py $c ${STEPS:-24} > $out/${tool}_$c.log 2>&1
    rc=$?
    echo "$tool $c rc=$rc $(( $(date +%s) - start ))s $(grep -E 'ERROR SUMMARY|RACECHECK SUMMARY|hazard' $out/${tool}_$c.log | tail -1)" | tee -a $out/summary.txt
  done
done
