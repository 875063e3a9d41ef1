"""Top source lines by warp-stall samples from `ncu -i REP --page source --csv --print-source cuda,sass`
output (one kernel), with each line's leading stall reasons.   python tools/ncu_source_lines.py CSV [N]"""
import csv, sys
from collections import defaultdict
rows = list(csv.reader(open(sys.argv[1])))
n_top = int(sys.argv[2]) if len(sys.argv) > 2 else 25
hdr = next(r for r in rows if len(r) > 10 and r[0] == "Line No")
stall = [i for i, h in enumerate(hdr) if h.startswith("stall_") and "Not Issued" not in h]
iS, iE = 4, hdr.index("Instructions Executed")
fname, lines = "", []
for r in rows:
    if len(r) >= 2 and r[0] in ("File Path", "File Name"):
        fname = r[1].split("/")[-1]
        continue
    if len(r) != len(hdr) or not r[0].isdigit():
        continue
    try:
        s = int(r[iS]); e = int(r[iE])
    except ValueError:
        continue
    st = {hdr[i][6:]: int(r[i]) for i in stall if r[i].isdigit() and int(r[i]) > 0}
    lines.append((s, e, fname, int(r[0]), r[1].strip()[:80], st))
tot = sum(l[0] for l in lines)
print(f"total samples {tot}")
for s, e, f, ln, src, st in sorted(lines, key=lambda l: -l[0])[:n_top]:
    top = sorted(st.items(), key=lambda kv: -kv[1])[:3]
    print(f"{100 * s / tot:5.1f}% {f}:{ln:<5} exec {e:>10} {' '.join(f'{k}={v}' for k, v in top):40s} {src}")
