#!/bin/bash
# compute-sanitizer memcheck / racecheck / synccheck over every device code path at
# config-1 size (tools/sanitize_case.py); logs + one summary line per run under $OUT.
OUT=${OUT:-gpurun_out/sanitize}
CASES=${CASES:-"resident exact tiled flat vc twoway slab"}
TOOLS=${TOOLS:-"memcheck racecheck synccheck"}
mkdir -p "$OUT"
for c in $CASES; do
  for t in $TOOLS; do
    s=$(date +%s)
    timeout 900 compute-sanitizer --tool "$t" --print-limit 50 --error-exitcode 9 \
      python tools/sanitize_case.py "$c" > "$OUT/$c.$t.log" 2>&1
    rc=$?
    echo "$c $t rc=$rc $(( $(date +%s) - s ))s $(grep -E 'ERROR SUMMARY|RACECHECK SUMMARY' "$OUT/$c.$t.log" | tail -1)" | tee -a "$OUT/summary.txt"
  done
done
