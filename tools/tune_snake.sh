#!/bin/bash
# Snake-order (TLGPU_SNAKE) and item-plan sweep of the streaming CG loops on the BASELINE
# grids (tools/solve_tune.py).  One JSON line per setting into $OUT.
OUT=${OUT:-gpurun_out/tune_snake.jsonl}
mkdir -p "$(dirname "$OUT")"
run() { env "$@" python tools/solve_tune.py $CFG $LVL 4 >> "$OUT" 2>> "$OUT.err"; }
for spec in "cfg4 local" "cfg3 global" "cfg3 local"; do
  set -- $spec; CFG=$1; LVL=$2
  for sn in 0 1; do
    run TLGPU_SNAKE=$sn TLGPU_TILED=0
    for th in 4 6 8; do
      for tc in 4 7 14; do
        run TLGPU_SNAKE=$sn TLGPU_TILED_MIN=1 TLGPU_TH=$th TLGPU_TC=$tc TLGPU_VERBOSE=1
      done
    done
  done
done
CFG=cfg4; LVL=global
for sn in 0 1; do
  for tc in 3 5 8; do
    run TLGPU_SNAKE=$sn TLGPU_TC=$tc TLGPU_VERBOSE=1
  done
done
