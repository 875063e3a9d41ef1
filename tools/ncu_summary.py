"""Summarise ncu --set full captures into profiles/<name>_summary.csv with FIXED units (time in ms,
bytes in GB, whatever unit each capture's raw page used), optionally refreshing
profiles/ncu_traffic.json (mean DRAM bytes per tile-pass launch, the bench's roofline.traffic).

    python tools/ncu_summary.py OUT_PREFIX "label;label;..." REP [REP ...] [--traffic KERNEL]

Each REP is an .ncu-rep; launches are labelled in order across the reps (missing labels: the
kernel name).  Every value is converted with its own capture's unit row, so captures whose ncu
chose different units (us vs ms, MB vs GB) never share a column unconverted.
"""
import csv
import io
import json
import os
import subprocess
import sys

COLS = ["Kernel Name", "launch__grid_size", "launch__block_size", "gpu__time_duration.sum",
        "dram__bytes_read.sum", "dram__bytes_write.sum",
        "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
        "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active",
        "smsp__issue_active.avg.pct_of_peak_sustained_active", "sm__warps_active.avg.pct_of_peak_sustained_active",
        "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum", "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum",
        "smsp__inst_executed.sum", "launch__registers_per_thread"]
TIME = {"ns": 1e-6, "us": 1e-3, "usecond": 1e-3, "msecond": 1.0, "ms": 1.0, "s": 1e3, "second": 1e3,
        "nsecond": 1e-6}
BYTES = {"byte": 1e-9, "Kbyte": 1e-6, "Mbyte": 1e-3, "Gbyte": 1.0, "Tbyte": 1e3}


def rows_of(rep):
    raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    hdr, units, data = rows[0], rows[1], rows[2:]
    out = []
    for d in data:
        rec = {}
        for c in COLS:
            if c not in hdr:
                rec[c] = ""
                continue
            i = hdr.index(c)
            v, u = d[i], units[i]
            if u in TIME:
                v = f"{float(v.replace(',', '')) * TIME[u]:.6f}"
            elif u in BYTES:
                v = f"{float(v.replace(',', '')) * BYTES[u]:.6f}"
            rec[c] = v
        out.append(rec)
    return out


def main():
    args = sys.argv[1:]
    traffic = None
    if "--traffic" in args:
        k = args.index("--traffic")
        traffic = args[k + 1]
        del args[k:k + 2]
    out, labels, reps = args[0], args[1].split(";") if args[1] else [], args[2:]
    recs = [r for rep in reps for r in rows_of(rep)]
    heads = ["pass"] + [c + ("[ms]" if c == "gpu__time_duration.sum" else "[GB]" if c.startswith("dram__bytes")
                             else "") for c in COLS] + ["achieved_GB/s"]
    with open(out + "_summary.csv", "w", newline="") as f:
        w = csv.writer(f)
        w.writerow(heads)
        for k, r in enumerate(recs):
            lab = labels[k] if k < len(labels) else r["Kernel Name"][:40]
            gbs = ""
            try:
                gbs = f"{(float(r['dram__bytes_read.sum']) + float(r['dram__bytes_write.sum'])) / float(r['gpu__time_duration.sum']) * 1e3:.1f}"
            except (ValueError, ZeroDivisionError):
                pass
            w.writerow([lab] + [r[c] for c in COLS] + [gbs])
    if traffic:
        tr = [(float(r["dram__bytes_read.sum"]) + float(r["dram__bytes_write.sum"])) * 1e9 for r in recs
              if traffic in r["Kernel Name"]]
        path = os.path.join(os.path.dirname(out), "ncu_traffic.json")
        json.dump({"tile": sum(tr) / len(tr), "per_launch": tr,
                   "source": f"{os.path.basename(out)}_summary.csv: ncu --set full --clock-control none, mean "
                             "dram__bytes_read.sum + dram__bytes_write.sum per launch"}, open(path, "w"), indent=1)
    print(open(out + "_summary.csv").read())


if __name__ == "__main__":
    main()
