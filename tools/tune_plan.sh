#!/bin/bash
# Item-plan check of k_t_cg (tools/solve_tune.py): the planner's default against explicit
# (TLGPU_TH, TLGPU_TC) neighbours on the BASELINE grids.  One JSON line per setting into $OUT.
OUT=${OUT:-gpurun_out/tune_plan.jsonl}
mkdir -p "$(dirname "$OUT")"; rm -f "$OUT" "$OUT.err"
run() { env TLGPU_VERBOSE=1 "$@" python tools/solve_tune.py $CFG $LVL 4 >> "$OUT" 2>> "$OUT.err"; }
CFG=cfg4; LVL=local;  run A=0; run TLGPU_TH=4 TLGPU_TC=14; run TLGPU_TH=4 TLGPU_TC=2; run TLGPU_TH=2 TLGPU_TC=7; run TLGPU_TILED=0
CFG=cfg3; LVL=global; run A=0; run TLGPU_TH=3 TLGPU_TC=7; run TLGPU_TH=3 TLGPU_TC=13; run TLGPU_TH=2 TLGPU_TC=6; run TLGPU_TILED=0
CFG=cfg3; LVL=local;  run A=0; run TLGPU_TH=6 TLGPU_TC=5; run TLGPU_TH=5 TLGPU_TC=19; run TLGPU_TH=6 TLGPU_TC=17; run TLGPU_TH=3 TLGPU_TC=3; run TLGPU_TILED=0
CFG=cfg4; LVL=global; run A=0; run TLGPU_TC=2; run TLGPU_TC=3; run TLGPU_TC=5
