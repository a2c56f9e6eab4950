"""Print selected metrics of ncu --page raw CSV exports side by side.
usage: python tools/ncu_keys.py A_raw.csv [B_raw.csv ...] [--grep regex]"""
import csv
import re
import sys

args = [a for a in sys.argv[1:] if not a.startswith("--grep")]
pat = re.compile(next((a.split("=", 1)[1] for a in sys.argv[1:] if a.startswith("--grep=")),
                      r"gpu__time_duration.sum$|smsp__issue_active.avg.pct|wavefronts_mem_shared.sum$|"
                      r"warp_issue_stalled_.*_per_warp_active.pct$|smsp__inst_executed.sum$|"
                      r"sm__warps_active.avg.pct|dram__bytes_read.sum$|pipe_(alu|fp64|lsu|xu|fma).*active.avg.pct_of_peak_sustained_active$|"
                      r"data_bank_conflicts.*sum$"))
tabs = []
for f in args:
    rows = list(csv.reader(open(f)))
    tabs.append({n: (rows[2][i], rows[1][i]) for i, n in enumerate(rows[0])})
names = [n for n in tabs[0] if pat.search(n)]
for n in names:
    vals = [t.get(n, ("-", ""))[0] for t in tabs]
    try:
        if all(float(v.replace(",", "")) == 0 for v in vals):
            continue
    except ValueError:
        pass
    print(f"{n[:90]:90s} " + " | ".join(f"{v:>14s}" for v in vals) + f"  {tabs[0].get(n, ('', ''))[1]}")
