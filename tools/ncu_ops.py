"""Per-opcode executed-instruction counts (per unit of work) from an ncu report's SASS source page."""
import collections
import csv
import subprocess
import sys

rep, units = sys.argv[1], float(sys.argv[2])
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                     capture_output=True, text=True).stdout.splitlines()
rows = list(csv.reader(out))
h = rows[1]
ie, src = h.index("Instructions Executed"), h.index("Source")
st = h.index("Warp Stall Sampling (All Samples)")
ops, stalls, tot = collections.Counter(), collections.Counter(), 0
for r in rows[2:]:
    try:
        n = int(r[ie])
    except (ValueError, IndexError):
        continue
    t = r[src].split()
    if not t:
        continue
    op = t[1] if t[0].startswith("@") else t[0]
    ops[op] += n
    stalls[op] += int(r[st] or 0)
    tot += n
print(f"thread-instructions per unit: {tot * 32 / units:.2f}")
for op, n in ops.most_common(int(sys.argv[3]) if len(sys.argv) > 3 else 25):
    print(f"{op:26s} {n * 32 / units:7.2f}   stall samples {stalls[op]}")
