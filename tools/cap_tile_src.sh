#!/bin/bash
# ncu --set full source-level captures (SASS per-instruction stalls and shared-memory wavefronts) of the
# cfg4 layer-boundary tile pass (second evaluation, skip 9) and the init pass (skip 7); output gpurun_out/diag/.
O=gpurun_out/diag; mkdir -p $O
python tools/prof_x.py 30 2 > /dev/null 2>&1
ncu --set full --clock-control none --import-source on -k regex:tile_pass -s 9 -c 1 -o /tmp/xb python tools/prof_x.py 30 2 > $O/xb.log 2>&1
ncu -i /tmp/xb.ncu-rep --page source --csv --print-source cuda > $O/xb_cuda.csv 2>/dev/null
ncu -i /tmp/xb.ncu-rep --page source --csv --print-source sass > $O/xb_sass.csv 2>/dev/null
ncu -i /tmp/xb.ncu-rep --page raw --csv > $O/xb_raw.csv 2>/dev/null
python tools/prof_x.py 30 2 > /dev/null 2>&1
ncu --set full --clock-control none --import-source on -k regex:tile_pass -s 7 -c 1 -o /tmp/xi python tools/prof_x.py 30 2 > $O/xi.log 2>&1
ncu -i /tmp/xi.ncu-rep --page source --csv --print-source cuda > $O/xi_cuda.csv 2>/dev/null
ls -la $O; head -c 600 $O/xb_cuda.csv
