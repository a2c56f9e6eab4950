"""Summarise ncu --set full reports into a markdown table (and the bench's traffic JSON).

usage: python tools/ncu_summary.py OUT.md [--traffic profiles/ncu_traffic.json[@KEY=trace:a,route:b,eval:c]...] name=report.ncu-rep[:units] ...
(each --traffic spec writes the named launches under workload KEY; default C5 = trace, route, eval)
`units` (optional) = requests / records / candidates processed by that launch,
to print instructions and DRAM bytes per unit."""
import csv
import json
import subprocess
import sys

KEYS = {
    "gpu__time_duration.sum": "duration",
    "dram__bytes_read.sum": "dram_read",
    "dram__bytes_write.sum": "dram_write",
    "dram__throughput.avg.pct_of_peak_sustained_elapsed": "dram_pct",
    "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed": "dram_pct",
    "sm__warps_active.avg.pct_of_peak_sustained_active": "occupancy_pct",
    "smsp__issue_active.avg.pct_of_peak_sustained_active": "issue_pct",
    "launch__registers_per_thread": "regs",
    "launch__grid_size": "grid",
    "launch__block_size": "block",
    "smsp__inst_executed.sum": "warp_inst",
    "sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active": "fp64_pipe_pct",
    "sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active": "alu_pipe_pct",
    "sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active": "lsu_pipe_pct",
}
UNIT_SCALE = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "Tbyte": 1e12,
              "nsecond": 1e-9, "usecond": 1e-6, "msecond": 1e-3, "second": 1.0,
              "ns": 1e-9, "us": 1e-6, "ms": 1e-3, "s": 1.0}


def raw(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(out.splitlines()))
    head, units, vals = rows[0], rows[1], rows[2]
    d = {}
    stalls = {}
    for i, n in enumerate(head):
        try:
            v = float(vals[i].replace(",", ""))
        except ValueError:
            continue
        v *= UNIT_SCALE.get(units[i], 1.0)
        if n in KEYS:
            d[KEYS[n]] = v
        if n.startswith("smsp__average_warps_issue_stalled_") and n.endswith("_per_issue_active.ratio"):
            stalls[n[len("smsp__average_warps_issue_stalled_"):-len("_per_issue_active.ratio")]] = v
    d["kernel"] = vals[head.index("Kernel Name")] if "Kernel Name" in head else "?"
    d["stalls"] = sorted(((k, v) for k, v in stalls.items() if k not in ("selected",)), key=lambda x: -x[1])[:3]
    return d


def main():
    out = sys.argv[1]
    args = sys.argv[2:]
    traffic_specs = []
    while args and args[0] == "--traffic":
        traffic_specs.append(args[1])
        args = args[2:]
    lines = ["| launch | kernel | µs | DRAM read GB | DRAM write GB | DRAM % of peak | occupancy % | issue % | "
             "regs | grid×block | instr/unit | bytes/unit | top stalls (warps per issue) |",
             "|---|---|---|---|---|---|---|---|---|---|---|---|---|"]
    traffic = {}
    for a in args:
        name, rest = a.split("=", 1)
        rep, units = (rest.split(":") + [None])[:2]
        d = raw(rep)
        u = float(units) if units else None
        ipu = d.get("warp_inst", 0) * 32 / u if u else None
        bpu = (d.get("dram_read", 0) + d.get("dram_write", 0)) / u if u else None
        lines.append(
            f"| {name} | `{d['kernel'][:60]}` | {d.get('duration', 0) * 1e6:.1f} | {d.get('dram_read', 0) / 1e9:.3f} | "
            f"{d.get('dram_write', 0) / 1e9:.3f} | {d.get('dram_pct', 0):.1f} | {d.get('occupancy_pct', 0):.1f} | "
            f"{d.get('issue_pct', 0):.1f} | {int(d.get('regs', 0))} | {int(d.get('grid', 0))}×{int(d.get('block', 0))} | "
            f"{'' if ipu is None else f'{ipu:.1f}'} | {'' if bpu is None else f'{bpu:.2f}'} | "
            + ", ".join(f"{k} {v:.2f}" for k, v in d["stalls"]) + " |")
        traffic[name] = {"dram_bytes_per_launch": d.get("dram_read", 0) + d.get("dram_write", 0),
                         "read": d.get("dram_read", 0), "write": d.get("dram_write", 0),
                         "ncu_duration_us": d.get("duration", 0) * 1e6}
    with open(out, "w") as f:
        f.write("\n".join(lines) + "\n")
    print("\n".join(lines))
    for spec in traffic_specs:
        path, _, rest = spec.partition("@")
        key, mapping = "C5", {"trace": "trace", "route": "route", "eval": "eval"}
        if rest:
            key, _, m = rest.partition("=")
            mapping = dict(kv.split(":") for kv in m.split(","))
        with open(path) as f:
            t = json.load(f)
        t[key] = {k: traffic[v] for k, v in mapping.items() if v in traffic}
        with open(path, "w") as f:
            json.dump(t, f, indent=1)


if __name__ == "__main__":
    main()
