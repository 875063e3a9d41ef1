#!/bin/bash
# A/B of environment switches on one box: per-evaluation tile-pass time (profiling events, repeated
# cfg4 evaluation, tools/pass_times.py) and the default bench step for each setting given.
for e in "$@"; do
    echo "== $e"
    env $e QVA_TRACE=1 python tools/pass_times.py 2>&1 | grep -E "^\[qva\] class|tile passes" | tail -9 | awk '/class/ {printf "%s ", $4} /tile passes/ {print ""; print}' 
    env $e python bench.py --no-cpu-baseline --steps 10 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.readline()); print('bench ms/step', round(d['ms_per_step'],3), 'e2e', round(d['e2e']['ms_per_step'],3), 'sm_mhz', d['clocks']['sm_mhz'])"
done
