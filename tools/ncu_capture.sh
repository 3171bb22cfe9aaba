#!/bin/bash
# One `ncu --set full` capture of the first k_t_cg launch of a solve, summarised on the GPU
# box (the .ncu-rep files are too large to bring back together): headline metrics, DRAM
# bytes, top source lines by stall samples.   tools/ncu_capture.sh cfg4 global [kernel-regex]
CFG=$1; LVL=$2; K=${3:-k_t_cg}; TAG=${TAG:-r02}
OUT=gpurun_out/${TAG}_${CFG}_${LVL}_${K}_ncu_full.txt
REP=/tmp/${TAG}_${CFG}_${LVL}_${K}
python tools/solve_once.py $CFG $LVL 1 > /dev/null 2>&1 || { echo "solve failed"; exit 1; }
ncu --set full --clock-control none --import-source on -k regex:$K -c 1 -f -o $REP python tools/solve_once.py $CFG $LVL 1 > gpurun_out/ncu_${CFG}_${LVL}.log 2>&1
{
  echo "# ncu --set full --clock-control none --import-source on -k regex:$K -c 1 python tools/solve_once.py $CFG $LVL 1"
  grep -E "rep 0" gpurun_out/ncu_${CFG}_${LVL}.log
  ncu -i $REP.ncu-rep --page raw --csv 2>/dev/null | python -c "
import csv,sys
rows=list(csv.reader(sys.stdin))
h=rows[0]; u=rows[1]; v=rows[2]
want=['dram__bytes_read.sum','dram__bytes_write.sum','gpu__time_duration.sum','lts__t_bytes.sum','l1tex__m_xbar2l1tex_read_bytes.sum','smsp__inst_executed.sum','sm__throughput.avg.pct_of_peak_sustained_elapsed','lts__t_sectors_srcunit_tex_op_read.sum','lts__t_sectors_op_write.sum','lts__t_sector_hit_rate.pct']
for k in want:
    if k in h:
        i=h.index(k); print('#', k, v[i], u[i])
"
  python tools/ncu_lines.py $REP.ncu-rep 28
} > $OUT 2>&1
if [ -n "$KEEP" ]; then cp $REP.ncu-rep gpurun_out/; fi
