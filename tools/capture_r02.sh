#!/bin/bash
# Round-2 evidence set (one gpurun call): bench lines, reference arm, ncu launch list of the default
# bench, ncu --set full summaries (cfg4 tile passes, cfg3 / 12! FFT passes, QAOAz tile passes).
set -u
V=${1:-v2}
O=gpurun_out
python bench.py > $O/r02_bench_default_$V.json 2> $O/r02_bench_default_$V.err
bash tools/bench_all.sh; cp $O/bench_all.jsonl $O/r02_bench_all_$V.jsonl
python bench.py --impl reference --steps 2 --warmup 3 > $O/r02_bench_reference_$V.json 2>&1
python tools/time_parity.py > $O/r02_qaoaz_timing_$V.txt 2>&1
python tools/time_qwoa.py 3 > $O/r02_qwoa_timing_$V.txt 2>&1
python tools/time_hostq.py > $O/r02_hostq_timing_$V.txt 2>&1 || true
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/r02_launches_qwoa12_$V.csv python tools/prof_qwoa12.py > /dev/null 2>&1
# launch list of the default bench (short run; plain run first)
python bench.py --steps 2 --warmup 3 --no-cpu-baseline > $O/plain_bench.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file $O/r02_launches_$V.csv \
    python bench.py --steps 2 --warmup 3 --no-cpu-baseline > $O/ncu_launch.log 2>&1
# --set full captures (plain runs first)
python tools/prof_x.py 30 1 > $O/plain_x.log 2>&1 && \
ncu --set full --clock-control none -k regex:tile_pass -c 7 -o /tmp/x python tools/prof_x.py 30 1 > $O/ncu_x.log 2>&1
python tools/prof_fft.py > $O/plain_fft.log 2>&1 && \
ncu --set full --clock-control none -k regex:fs_ -c 9 -o /tmp/fft3 python tools/prof_fft.py > $O/ncu_fft3.log 2>&1
python tools/prof_qwoa12.py > $O/plain_q12.log 2>&1 && \
ncu --set full --clock-control none -k regex:fs_ -c 5 -o /tmp/fft12 python tools/prof_qwoa12.py > $O/ncu_fft12.log 2>&1
python tools/prof_parity.py > $O/plain_par.log 2>&1 && \
ncu --set full --clock-control none -k regex:tile_pass -c 6 -o /tmp/par python tools/prof_parity.py > $O/ncu_par.log 2>&1
python tools/ncu_summary.py $O/r02_ncu_tile_cfg4_$V "init P|XY;A XWY;B XY|P|YX;A XWY;B XY|P|YX;A XWY;C XY+<Q>" /tmp/x.ncu-rep --traffic tile_pass > /dev/null
python tools/ncu_summary.py $O/r02_ncu_fft_$V "" /tmp/fft3.ncu-rep /tmp/fft12.ncu-rep > /dev/null
python tools/ncu_summary.py $O/r02_ncu_parity_$V "" /tmp/par.ncu-rep > /dev/null
cp $O/ncu_traffic.json $O/ncu_traffic_$V.json 2>/dev/null
ls -la $O | tail -30
