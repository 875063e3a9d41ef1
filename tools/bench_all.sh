#!/bin/bash
# One bench line per workload (device-timed value, roofline of the dominant kernel, e2e where the
# workload has one); output: gpurun_out/bench_all.jsonl
set -u
out=gpurun_out/bench_all.jsonl
: > $out
for w in cfg1 cfg2 cfg3 cfg3cf cfg4 cfg5w qaoaz28 qwoa12; do
    steps=10; [ $w = qwoa12 ] && steps=3
    python bench.py --workload $w --no-cpu-baseline --steps $steps >> $out 2>> gpurun_out/bench_all.err || echo "{\"workload\": \"$w\", \"failed\": true}" >> $out
done
