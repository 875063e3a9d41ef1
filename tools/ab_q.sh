#!/bin/bash
# per-pass times (ncu launch list, cold) of one cfg4 evaluation: generated vs stored (int8) q
for mode in gen stored gen; do
    python tools/prof_x.py 30 1 $mode > /dev/null 2>&1 && ncu --metrics gpu__time_duration.sum --clock-control none -k regex:tile_pass --csv --log-file /tmp/l.csv python tools/prof_x.py 30 1 $mode > /dev/null 2>&1
    echo "== $mode: $(grep tile_pass /tmp/l.csv | awk -F, '{gsub(/"/,"",$NF); s+=$NF; printf "%.3f ", $NF/1e6} END {printf " sum %.3f ms", s/1e6}')"
done
