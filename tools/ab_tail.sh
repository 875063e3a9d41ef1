#!/bin/bash
# A/B of measurement switches on one box: per-pass times (ncu launch list, cold) of one cfg4
# evaluation for each environment setting given as arguments.
for e in "$@"; do
    env $e python tools/prof_x.py 30 1 > /dev/null 2>&1 && env $e ncu --metrics gpu__time_duration.sum --clock-control none -k regex:tile_pass --csv --log-file /tmp/l.csv python tools/prof_x.py 30 1 > /dev/null 2>&1
    echo "== $e: $(grep tile_pass /tmp/l.csv | awk -F, '{gsub(/"/,"",$NF); s+=$NF; printf "%.3f ", $NF/1e6} END {printf " sum %.3f ms", s/1e6}')"
done
