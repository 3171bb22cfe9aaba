#!/bin/bash
# Default-plan solve times of the four streaming grids (tools/solve_tune.py), one JSON line each.
OUT=${OUT:-gpurun_out/tune_quick.jsonl}
mkdir -p "$(dirname "$OUT")"; rm -f "$OUT" "$OUT.err"
for spec in "cfg4 local" "cfg3 global" "cfg3 local" "cfg4 global"; do
  set -- $spec
  TLGPU_VERBOSE=1 python tools/solve_tune.py $1 $2 4 >> "$OUT" 2>> "$OUT.err"
done
