#!/bin/bash
# Solver-path sweep on the local grids (tools/solve_tune.py): flat k_s_cg vs the bulk-copy
# z-march k_t_cg at several item shapes.  One JSON line per setting into $OUT.
OUT=${OUT:-gpurun_out/tune_local.jsonl}
mkdir -p "$(dirname "$OUT")"
for c in ${CFGS:-cfg4 cfg3}; do
  python tools/solve_tune.py $c local 4 >> "$OUT" 2>&1
  for th in ${THS:-2 4 6}; do
    for tz in ${TZS:-3 8 16}; do
      TLGPU_TILED_MIN=1 TLGPU_TH=$th TLGPU_TZ=$tz python tools/solve_tune.py $c local 4 >> "$OUT" 2>&1
    done
  done
done
