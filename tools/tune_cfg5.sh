#!/bin/bash
OUT=gpurun_out/tune_cfg5.txt; rm -f $OUT
run() { echo "== $*" >> $OUT; env TLGPU_VERBOSE=1 "$@" python bench.py --config cfg5 --steps 4 --warmup 3 --no-cpu-baseline > /tmp/b5.json 2> /tmp/b5.err; grep "item plan" /tmp/b5.err | sort | uniq -c | head -4 >> $OUT; python - >> $OUT <<PY
import json
for l in open("/tmp/b5.json"):
    if l.startswith("{"):
        d=json.loads(l); k=d["kernels"]; print(d["ms_per_step"], k["local_pcg"]["avg_ms_per_solve"], k["local_pcg"]["achieved_gbs"], k["global_pcg"]["avg_ms_per_solve"], k["global_pcg"]["achieved_gbs"])
PY
}
run A=0
run TLGPU_TH=12 TLGPU_TC=1 TLGPU_NCW=19
run TLGPU_TH=10 TLGPU_TC=3 TLGPU_NCW=16
run TLGPU_TH=5 TLGPU_TC=2 TLGPU_NCW=16
run TLGPU_TH=6 TLGPU_TC=1 TLGPU_NCW=19
run TLGPU_TH=3 TLGPU_TC=1 TLGPU_NCW=19
run TLGPU_TH=6 TLGPU_TC=5 TLGPU_NCW=19
cat $OUT
