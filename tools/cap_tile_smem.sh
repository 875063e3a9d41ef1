#!/bin/bash
# ncu --set full of the second cfg4 evaluation's first three tile passes (init P|XY, window XWY,
# layer boundary XY|P|YX): raw page rows of the shared-memory / L1 data-pipe utilisation metrics
# next to duration, DRAM and fp64 figures.  Output gpurun_out/diag/tile_smem_raw.csv and
# gpurun_out/diag/tile_smem_pipes.txt (metric name, unit, one value per launch).
O=gpurun_out/diag; mkdir -p $O
python tools/prof_x.py 30 2 > /dev/null 2>&1 || exit 1
ncu --set full --clock-control none -k regex:tile_pass -s 7 -c 3 -o /tmp/xs python tools/prof_x.py 30 2 > $O/xs.log 2>&1
ncu -i /tmp/xs.ncu-rep --page raw --csv > $O/tile_smem_raw.csv 2>/dev/null
python - <<'EOF'
import csv
rows = list(csv.reader(open("gpurun_out/diag/tile_smem_raw.csv")))
hdr, units, data = rows[0], rows[1], rows[2:]
keys = ("Kernel Name", "gpu__time_duration.sum", "sm__cycles_elapsed.avg", "sm__cycles_active.avg",
        "l1tex__data_pipe", "l1tex__data_bank", "l1tex__throughput", "l1tex__lsu_writeback", "smsp__inst_executed_pipe_lsu",
        "sm__inst_executed_pipe_lsu", "sm__mio", "smsp__mio", "sm__pipe_fp64", "dram__throughput", "gpu__dram_throughput",
        "l1tex__m_xbar2l1tex", "l1tex__m_l1tex2xbar", "smem", "shared", "sm__throughput", "l1tex__t_")
with open("gpurun_out/diag/tile_smem_pipes.txt", "w") as f:
    for i, h in enumerate(hdr):
        if any(k in h for k in keys):
            f.write(f"{h} [{units[i]}]: " + " | ".join(d[i] for d in data) + "\n")
EOF
wc -l $O/tile_smem_pipes.txt
