#!/bin/bash
# cfg2 batch tile passes: per-launch metrics of one batch evaluation and --set full captures with
# source of the init and boundary passes.  Output under gpurun_out/dcfg2/.
O=gpurun_out/dcfg2; mkdir -p $O
python tools/prof_cfg2.py > /dev/null 2>&1
M=gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,smsp__issue_active.avg.pct_of_peak_sustained_active,sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active,smsp__inst_executed.sum
ncu --metrics $M --clock-control none -k regex:tile_pass -s 6 -c 6 --csv python tools/prof_cfg2.py > $O/metrics.csv 2>&1
for spec in "init 6" "bnd 8"; do set -- $spec
  ncu --set full --clock-control none --import-source on -k regex:tile_pass -s $2 -c 1 -o /tmp/c2$1 python tools/prof_cfg2.py > $O/$1.log 2>&1
  ncu -i /tmp/c2$1.ncu-rep --page source --csv --print-source cuda,sass > /tmp/c2$1.csv 2>/dev/null
  python tools/ncu_source_lines.py /tmp/c2$1.csv 30 > $O/$1_lines.txt 2>&1
done
