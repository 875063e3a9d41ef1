#!/bin/bash
# Diagnostic set (one gpurun call): per-pass A/B of store modes on cfg4, and ncu --set full
# captures with source (stall reasons per line) of the cfg4 init / boundary passes and of the
# 12! / cfg3 FFT row and column kernels.  Output under gpurun_out/diag/.
set -u
O=gpurun_out/diag; mkdir -p $O
bash tools/ab_tail.sh "QVA_TSTORE=1" "QVA_TSTORE=0" "QVA_TAIL=2" > $O/ab_store.txt 2>&1
cap() {  # name, kernel regex, skip, driver...
    local n=$1 k=$2 s=$3; shift 3
    ncu --set full --clock-control none --import-source on -k regex:$k -s $s -c 1 -o /tmp/$n "$@" > $O/$n.log 2>&1
    ncu -i /tmp/$n.ncu-rep --page source --csv --print-source cuda,sass > $O/${n}_src.csv 2>/dev/null
    python tools/ncu_source_lines.py $O/${n}_src.csv 40 > $O/${n}_lines.txt 2>&1
    ncu -i /tmp/$n.ncu-rep --page raw --csv > $O/${n}_raw.csv 2>/dev/null
    rm -f $O/${n}_src.csv
}
python tools/prof_x.py 30 2 > /dev/null 2>&1
cap x_init tile_pass 7 python tools/prof_x.py 30 2
cap x_bnd tile_pass 9 python tools/prof_x.py 30 2
python tools/prof_qwoa12.py > /dev/null 2>&1
cap q12_row fft_row 0 python tools/prof_qwoa12.py
cap q12_col2 fft_col 1 python tools/prof_qwoa12.py
cap q12_col1 fft_col 0 python tools/prof_qwoa12.py
cap c3_row fft_row 1 python tools/prof_fft.py
cap c3_col fft_col 1 python tools/prof_fft.py
ls -la $O
