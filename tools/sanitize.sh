#!/bin/bash
# compute-sanitizer over tools/sanitize_driver.py (run under gpurun, one GPU):
# memcheck (incl. leak check), racecheck (shared-memory hazards), synccheck
# (barrier misuse) and initcheck (uninitialised global reads).  Summaries ->
# gpurun_out/sanitize_<tool>.log; the tail of each is committed under profiles/.
OUT=${OUT:-gpurun_out}
for tool in memcheck racecheck synccheck initcheck; do
  extra=""
  [ "$tool" = memcheck ] && extra="--leak-check full"
  SAN_TOOL=$tool timeout ${SAN_TIMEOUT:-1500} compute-sanitizer --tool $tool $extra --target-processes all \
    --print-limit 50 python tools/sanitize_driver.py > $OUT/sanitize_$tool.log 2>&1
  echo "$tool rc=$? $(grep -E 'ERROR SUMMARY|RACECHECK SUMMARY|LEAK SUMMARY' $OUT/sanitize_$tool.log | tr '\n' ' ')"
done
