#!/usr/bin/env python
"""Per-instruction stall attribution of an ncu --set full report (SASS view):
top instructions by samples with their dominant stall reasons, and the sample share
of instruction classes.  python tools/sass_hotspots.py rep.ncu-rep [--top 40]"""
import argparse
import collections
import csv
import io
import subprocess

p = argparse.ArgumentParser()
p.add_argument("rep")
p.add_argument("--top", type=int, default=40)
p.add_argument("--ranges", default="", help="comma list a-b of SASS line ranges to total")
a = p.parse_args()
out = subprocess.run(["ncu", "-i", a.rep, "--page", "source", "--csv", "--print-source", "sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
hdr, data = rows[1], rows[2:]
col = {h: i for i, h in enumerate(hdr)}
reasons = [h for h in hdr if h.startswith("stall_") and "Not Issued" not in h]
tot = sum(int(r[col["Warp Stall Sampling (All Samples)"]] or 0) for r in data)
print("total samples", tot)
cls = collections.Counter()
rs = collections.Counter()
for r in data:
    s = int(r[col["Warp Stall Sampling (All Samples)"]] or 0)
    op = r[col["Source"]].strip().split()
    op = [x for x in op if not x.startswith("@")]
    cls[op[0].split(".")[0] if op else "?"] += s
    for h in reasons:
        rs[h] += int(r[col[h]] or 0)
print("by class:", ", ".join(f"{k} {100 * v / tot:.1f}%" for k, v in cls.most_common(14)))
print("by reason:", ", ".join(f"{k[6:]} {100 * v / tot:.1f}%" for k, v in rs.most_common(10)))
top = sorted(range(len(data)), key=lambda k: -int(data[k][col["Warp Stall Sampling (All Samples)"]] or 0))[:a.top]
for k in sorted(top):
    r = data[k]
    s = int(r[col["Warp Stall Sampling (All Samples)"]] or 0)
    why = sorted(((int(r[col[h]] or 0), h[6:]) for h in reasons), reverse=True)[:2]
    print(f"{k:5d} {100 * s / tot:5.2f}% ex={r[col['Instructions Executed']]:>10} {r[col['Source']].strip()[:70]:70s} "
          + " ".join(f"{n}:{100 * v / max(s, 1):.0f}%" for v, n in why))
for rg in filter(None, a.ranges.split(",")):
    lo, hi = map(int, rg.split("-"))
    s = sum(int(data[k][col["Warp Stall Sampling (All Samples)"]] or 0) for k in range(lo, hi + 1))
    print(f"lines {lo}-{hi}: {100 * s / tot:.1f}% of samples")
