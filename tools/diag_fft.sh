#!/bin/bash
# FFT pass diagnostics (one gpurun call): per-launch metrics of one p=1 QWOA evolution at 12! and
# of the cfg3 evolution, and --set full captures with source of the fused-stage row / column
# kernels (stall reasons per line).  Output under gpurun_out/dfft/.
set -u
O=gpurun_out/dfft; mkdir -p $O
M=gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,smsp__issue_active.avg.pct_of_peak_sustained_active,sm__warps_active.avg.pct_of_peak_sustained_active,launch__registers_per_thread,smsp__inst_executed.sum,l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum,sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active,launch__grid_size,launch__block_size
python tools/prof_qwoa12.py > /dev/null 2>&1 && ncu --metrics $M --clock-control none -k regex:fs_ --csv python tools/prof_qwoa12.py > $O/q12_metrics.csv 2>&1
python tools/prof_fft.py > /dev/null 2>&1 && ncu --metrics $M --clock-control none -k regex:fs_ --csv python tools/prof_fft.py > $O/c3_metrics.csv 2>&1
cap() {  # name, kernel regex, skip, driver...
    local n=$1 k=$2 s=$3; shift 3
    ncu --set full --clock-control none --import-source on -k regex:$k -s $s -c 1 -o /tmp/$n "$@" > $O/$n.log 2>&1
    ncu -i /tmp/$n.ncu-rep --page source --csv --print-source cuda,sass > /tmp/${n}_src.csv 2>/dev/null
    python tools/ncu_source_lines.py /tmp/${n}_src.csv 40 > $O/${n}_lines.txt 2>&1
    ncu -i /tmp/$n.ncu-rep --page raw --csv > $O/${n}_raw.csv 2>/dev/null
}
for spec in ${FS_CAPS:-"q12_row fs_row 0 tools/prof_qwoa12.py" "q12_colA fs_col 1 tools/prof_qwoa12.py" "q12_colO fs_col 0 tools/prof_qwoa12.py"}; do
    set -- $spec
    cap $1 $2 $3 python $4
done
ls -la $O
