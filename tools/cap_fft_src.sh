#!/bin/bash
# ncu --set full source-level captures (SASS per-instruction stalls and shared-memory wavefronts) of the
# 12! three-level FFT inner row pass (fs_rowpp, 768-point rows) and inner column pass; output gpurun_out/diag/.
O=gpurun_out/diag; mkdir -p $O
python tools/prof_qwoa12.py > /dev/null 2>&1
ncu --set full --clock-control none --import-source on -k regex:fs_rowpp -s 20 -c 1 -o /tmp/frow python tools/prof_qwoa12.py > $O/frow.log 2>&1
ncu -i /tmp/frow.ncu-rep --page source --csv --print-source sass > $O/frow_sass.csv 2>/dev/null
ncu -i /tmp/frow.ncu-rep --page source --csv --print-source cuda > $O/frow_cuda.csv 2>/dev/null
ncu --set full --clock-control none --import-source on -k regex:fs_colpp -s 21 -c 1 -o /tmp/fcol python tools/prof_qwoa12.py > $O/fcol.log 2>&1
ncu -i /tmp/fcol.ncu-rep --page source --csv --print-source sass > $O/fcol_sass.csv 2>/dev/null
ls -la $O
