"""Summarise an ncu --set full capture of the X-mixer tile passes (tools/prof_x.py 30 1) into
profiles/<name>_summary.csv and refresh profiles/ncu_traffic.json (mean DRAM bytes per launch).

    python tools/ncu_summary.py gpurun_out/prof_tile_v5.ncu-rep profiles/r01_ncu_tile_v5 "pass labels;..."
"""
import csv, io, json, os, subprocess, sys

rep, out, labels = sys.argv[1], sys.argv[2], sys.argv[3].split(";")
raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(raw)))
hdr, units, data = rows[0], rows[1], rows[2:]
cols = ["Kernel Name", "gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
        "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active",
        "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum", "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum",
        "l1tex__throughput.avg.pct_of_peak_sustained_active", "smsp__issue_active.avg.pct_of_peak_sustained_active",
        "smsp__inst_executed.sum", "launch__registers_per_thread"]
idx = [hdr.index(c) for c in cols]
with open(out + "_summary.csv", "w", newline="") as f:
    w = csv.writer(f)
    w.writerow(["pass"] + [c + (f"[{units[i]}]" if units[i] else "") for c, i in zip(cols, idx)])
    for lab, d in zip(labels, data):
        w.writerow([lab] + [d[i] for i in idx])
scale = {"Gbyte": 1e9, "Mbyte": 1e6, "Kbyte": 1e3, "byte": 1.0}
ir, iw = hdr.index("dram__bytes_read.sum"), hdr.index("dram__bytes_write.sum")
tr = [float(d[ir]) * scale[units[ir]] + float(d[iw]) * scale[units[iw]] for d in data]
path = os.path.join(os.path.dirname(out), "ncu_traffic.json")
json.dump({"tile": sum(tr) / len(tr), "per_launch": tr,
           "source": f"{os.path.basename(out)}_summary.csv: ncu --set full --clock-control none of the "
                     f"{len(tr)} tile passes of one cfg4 evolve (tools/prof_x.py 30 1), mean "
                     "dram__bytes_read.sum + dram__bytes_write.sum per launch"},
          open(path, "w"), indent=1)
print(open(out + "_summary.csv").read())
print("traffic per launch (GB):", [round(x / 1e9, 3) for x in tr])
