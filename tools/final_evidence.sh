#!/bin/bash
mkdir -p gpurun_out/final
python -m pytest tests -m gpu -q 2>&1 | tail -25 > gpurun_out/final/gputest.log
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/final/smoke.log 2>&1
( time python bench.py ) > gpurun_out/final/bench_default.jsonl 2> gpurun_out/final/bench_default.err
( time python bench.py --impl reference ) > gpurun_out/final/bench_reference.jsonl 2> gpurun_out/final/bench_reference.err
python bench.py --config cfg2 --steps 20 --warmup 3 --no-cpu-baseline > gpurun_out/final/bench_cfg2.jsonl 2>/dev/null
python bench.py --config cfg3 --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/final/bench_cfg3.jsonl 2>/dev/null
python bench.py --config cfg5 --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/final/bench_cfg5.jsonl 2>/dev/null
python bench.py --slabs --no-cpu-baseline > gpurun_out/final/bench_slabs.jsonl 2>/dev/null
tail -3 gpurun_out/final/gputest.log; cat gpurun_out/final/smoke.log | tail -2
for f in default reference cfg2 cfg3 cfg5 slabs; do python - <<PY
import json
for l in open("gpurun_out/final/bench_$f.jsonl"):
    if l.startswith("{"):
        d=json.loads(l); print("$f", d.get("value"), d.get("ms_per_step"), (d.get("e2e") or {}).get("value"), (d.get("roofline") or {}).get("frac"), d.get("clocks",{}).get("reasons"))
PY
done
grep real gpurun_out/final/bench_default.err gpurun_out/final/bench_reference.err
