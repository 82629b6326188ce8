#!/bin/bash
# compute-sanitizer over every kernel family (SURVEY §5 / VERDICT r1 #4):
#   tools/sanitize.sh [tools...]      (default: memcheck racecheck synccheck)
# One small case per family (tools/sanitize_case.py), each bounded by `timeout`.
# Logs: gpurun_out/sanitize/<tool>_<case>.log; summary: gpurun_out/sanitize/summary.txt
# PYTORCH_NO_CUDA_MEMORY_CACHING=1: every torch tensor is its own allocation, so
# memcheck sees out-of-bounds accesses into torch-owned buffers too.
cd "$(dirname "$0")/.."
OUT=gpurun_out/sanitize
mkdir -p $OUT
TOOLS=${@:-memcheck racecheck synccheck}
CASES=${CASES:-$(python tools/sanitize_case.py list 2>/dev/null | sed 's/^cases: //')}
CS=/usr/local/cuda/bin/compute-sanitizer
$CS --version | head -2 > $OUT/version.txt
: > $OUT/summary.txt
for tool in $TOOLS; do
  for c in $CASES; do
    log=$OUT/${tool}_$c.log
    extra=""
    [ $tool = memcheck ] && extra="--leak-check no"
    [ $tool = racecheck ] && extra="--racecheck-report hazard"
    t0=$(date +%s)
    PYTORCH_NO_CUDA_MEMORY_CACHING=1 timeout ${SAN_TIMEOUT:-300} $CS --tool $tool $extra \
        --error-exitcode 99 python tools/sanitize_case.py $c > $log 2>&1
    rc=$?
    t1=$(date +%s)
    ok=$(grep -c " ok$" $log)
    summ=$(grep -E "ERROR SUMMARY|RACECHECK SUMMARY|Error|hazard" $log | tail -1)
    echo "$tool $c rc=$rc case_ok=$ok ${t1}-${t0}s :: $summ" | sed "s/${t1}-${t0}/$((t1-t0))/" >> $OUT/summary.txt
  done
done
cat $OUT/summary.txt
