"""SASS listing of a kernel's hot loop, with an instruction count per unit of work.

For each function matching --kernel, finds the backward branches (loops), picks the
loop body with the most instructions matching --marker (the hot loop's streaming
loads by default), prints it and a mnemonic histogram, and divides the instruction
count by --units (requests, records ... processed per thread per iteration).

Evidence for DESIGN.md §5's per-request instruction counts (the verdict asked for
the SASS behind them). Runs here, on the CPU: cuobjdump only.

  python tools/sass_hotloop.py --kernel 'k1_traceILi1ELi32ELb0ELb1ELb0ELb1ELb1E' --units 16
"""
from __future__ import annotations

import argparse
import collections
import os
import re
import signal
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
LIB = os.path.join(ROOT, "paper_2604_08075_b200", "lib", "libfleetplan.so")
INS = re.compile(r"/\*([0-9a-f]{4,})\*/\s+(.*?)\s*;")


def functions(lib):
    out = subprocess.run(["cuobjdump", "-sass", lib], check=True, capture_output=True, text=True).stdout
    funcs, name, body = {}, None, []
    for line in out.splitlines():
        if "Function :" in line:
            if name:
                funcs[name] = body
            name, body = line.split("Function :")[1].strip(), []
            continue
        m = INS.search(line)
        if name and m:
            body.append((int(m.group(1), 16), m.group(2).strip()))
    if name:
        funcs[name] = body
    return funcs


def loops(body):
    """(start, end) address ranges of backward branches."""
    res = []
    for addr, text in body:
        m = re.search(r"\bBRA(?:\.\S+)?\s+(?:\S+,\s*)?(0x[0-9a-f]+)", text)
        if m:
            tgt = int(m.group(1), 16)
            if tgt <= addr:
                res.append((tgt, addr))
    return res


def walk(body, lo, hi, take):
    """One iteration's instructions from the loop head: follow unconditional branches,
    decide conditional ones from `take`, stop at the back edge (a branch to lo)."""
    at = {ad: i for i, (ad, _) in enumerate(body)}
    i, k, path = at[lo], 0, []
    while i < len(body) and len(path) < 100000:
        ad, t = body[i]
        path.append((ad, t))
        m = re.search(r"\bBRA(?:\.\S+)?\s+(?:(!?U?P\w+),\s*)?(0x[0-9a-f]+)", t)
        if m:
            tgt = int(m.group(2), 16)
            cond = bool(m.group(1)) or t.startswith("@")
            if tgt == lo and ad == hi:
                break
            if not cond or (k < len(take) and take[k] == "t"):
                i = at[tgt]
            else:
                i += 1
            k += cond
            continue
        i += 1
    return path


def mnemonic(text):
    t = re.sub(r"^@!?U?P\w+\s+", "", text)
    return t.split()[0]


def main():
    signal.signal(signal.SIGPIPE, signal.SIG_DFL)
    ap = argparse.ArgumentParser()
    ap.add_argument("--kernel", required=True, help="substring of the mangled name")
    ap.add_argument("--marker", default=r"LDG\.E\S*\.128", help="regex counted to pick the hot loop")
    ap.add_argument("--units", type=float, default=1.0, help="work units per thread per loop iteration")
    ap.add_argument("--lib", default=LIB)
    ap.add_argument("--smallest", action="store_true",
                    help="pick the smallest loop containing the marker (nested loops) instead of the one "
                         "with the most marker hits")
    ap.add_argument("--listing", action="store_true", help="print the loop body")
    ap.add_argument("--take", default=None,
                    help="walk one iteration from the loop head instead of counting the whole loop "
                         "range: 't'/'n' per conditional branch met (taken / not taken; default n), "
                         "unconditional branches followed, stop at the back edge")
    a = ap.parse_args()
    for name, body in functions(a.lib).items():
        if a.kernel not in name:
            continue
        best = None
        for lo, hi in loops(body):
            ins = [(ad, t) for ad, t in body if lo <= ad <= hi]
            hits = sum(1 for _, t in ins if re.search(a.marker, t))
            key = (-len(ins), hits) if a.smallest else (hits, -len(ins))
            if hits and (best is None or key > best[4]):
                best = (hits, ins, lo, hi, key)
        print(f"== {name}")
        if best is None:
            print("   no loop containing the marker")
            continue
        hits, ins, lo, hi, _ = best
        if a.take is not None:
            ins = walk(body, lo, hi, a.take)
            hits = sum(1 for _, t in ins if re.search(a.marker, t))
        hist = collections.Counter(mnemonic(t) for _, t in ins)
        print(f"   hot loop 0x{lo:x}..0x{hi:x}: {len(ins)} instructions, {hits} marker hits, "
              f"{len(ins) / a.units:.2f} instructions per unit ({a.units:g} units/iteration)")
        for k, v in sorted(hist.items(), key=lambda kv: -kv[1]):
            print(f"   {v:5d}  {k}")
        if a.listing:
            for ad, t in ins:
                print(f"   /*{ad:04x}*/ {t}")
    return 0


if __name__ == "__main__":
    sys.exit(main())
