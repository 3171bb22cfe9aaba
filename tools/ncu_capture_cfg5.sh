#!/bin/bash
REP=/tmp/r02_cfg5_k_tb_cg
ncu --set full --clock-control none --import-source on -k regex:k_tb_cg -s 20 -c 1 -f -o $REP python bench.py --config cfg5 --steps 1 --warmup 3 --no-cpu-baseline > gpurun_out/ncu_cfg5.log 2>&1
{
  echo "# ncu --set full --clock-control none --import-source on -k regex:k_tb_cg -s 20 -c 1 python bench.py --config cfg5 --steps 1 --warmup 3"
  ncu -i $REP.ncu-rep --page raw --csv 2>/dev/null | python -c "
import csv,sys
rows=list(csv.reader(sys.stdin))
h=rows[0]; u=rows[1]; v=rows[2]
want=['dram__bytes_read.sum','dram__bytes_write.sum','gpu__time_duration.sum','lts__t_bytes.sum','l1tex__m_xbar2l1tex_read_bytes.sum','smsp__inst_executed.sum','sm__throughput.avg.pct_of_peak_sustained_elapsed','lts__t_sector_hit_rate.pct','launch__grid_size','launch__block_size']
for k in want:
    if k in h:
        i=h.index(k); print('#', k, v[i], u[i])
"
  python tools/ncu_lines.py $REP.ncu-rep 30
} > gpurun_out/r02_cfg5_k_tb_cg_ncu_full.txt 2>&1
head -50 gpurun_out/r02_cfg5_k_tb_cg_ncu_full.txt
