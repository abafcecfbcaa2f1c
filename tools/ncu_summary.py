#!/usr/bin/env python
"""Summarise ncu evidence for profiles/: a --set full report of the top kernel and a
--metrics gpu__time_duration.sum launch list (both captured under gpurun).

  python tools/ncu_summary.py --rep gpurun_out/prof.ncu-rep [--launches gpurun_out/launches.csv] > profiles/x.md
  python tools/ncu_summary.py --rep ... --traffic-json profiles/ncu_traffic_c2.json
"""
from __future__ import annotations

import argparse
import collections
import csv
import json
import subprocess

KEYS = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "lts__throughput.avg.pct_of_peak_sustained_elapsed",
        "lts__t_sector_hit_rate.pct", "l1tex__throughput.avg.pct_of_peak_sustained_active",
        "sm__throughput.avg.pct_of_peak_sustained_elapsed", "smsp__issue_active.avg.pct_of_peak_sustained_active",
        "sm__warps_active.avg.pct_of_peak_sustained_active", "smsp__warps_eligible.avg.per_cycle_active",
        "smsp__inst_executed.sum", "launch__registers_per_thread", "launch__grid_size", "launch__block_size",
        "launch__shared_mem_per_block_dynamic", "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active"]

SCALE = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "Tbyte": 1e12}


def raw(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    r = list(csv.reader(out.splitlines()))
    return r[0], r[1], r[2:]


def kernel_sha16() -> str:
    """Hash of the K1 sources (bench.py compares it to decide whether a capture is current)."""
    import hashlib
    from pathlib import Path

    csrc = Path(__file__).resolve().parents[1] / "paper_1606_07822_b200" / "csrc"
    h = hashlib.sha256()
    for name in ("cg_hogwild.cu", "cg_hog8.cu", "cg_device.cuh"):
        if (csrc / name).exists():
            h.update((csrc / name).read_bytes())
    return h.hexdigest()[:16]


def to_bytes(v, unit):
    return float(v.replace(",", "")) * SCALE.get(unit, 1)


def main():
    p = argparse.ArgumentParser()
    p.add_argument("--rep", required=True)
    p.add_argument("--launches")
    p.add_argument("--traffic-json")
    p.add_argument("--title", default="")
    a = p.parse_args()
    h, units, rows = raw(a.rep)
    name_i = h.index("Kernel Name")
    print(f"# ncu summary {a.title}\n\nreport: `{a.rep}`\n")
    for row in rows:
        print(f"## {row[name_i][:100]}\n")
        print("| metric | value | unit |\n|---|---|---|")
        for k in KEYS:
            if k in h:
                i = h.index(k)
                print(f"| {k} | {row[i]} | {units[i]} |")
        st = [(h[i], row[i]) for i in range(len(h)) if h[i].startswith("smsp__pcsamp_warps_issue_stalled")
              and not h[i].endswith("not_issued")]
        tot = sum(float(x or 0) for _, x in st) or 1.0
        print("\nwarp stall samples (share):\n")
        for k, x in sorted(st, key=lambda t: -float(t[1] or 0))[:8]:
            print(f"- {k.replace('smsp__pcsamp_warps_issue_stalled_', '')}: {float(x) / tot * 100:.1f}%")
        rd = to_bytes(row[h.index("dram__bytes_read.sum")], units[h.index("dram__bytes_read.sum")])
        wr = to_bytes(row[h.index("dram__bytes_write.sum")], units[h.index("dram__bytes_write.sum")])
        print(f"\nDRAM traffic per launch: {rd + wr:.4g} bytes (read {rd:.4g}, write {wr:.4g})")
        l2 = None
        if "lts__t_sectors.sum" in h:
            l2 = float(row[h.index("lts__t_sectors.sum")].replace(",", "")) * 32.0
            t_ms = float(row[h.index("gpu__time_duration.sum")].replace(",", ""))
            t_s = t_ms * {"s": 1.0, "second": 1.0, "ms": 1e-3, "msecond": 1e-3, "us": 1e-6, "usecond": 1e-6, "ns": 1e-9, "nsecond": 1e-9}.get(
                units[h.index("gpu__time_duration.sum")], 1e-3)
            print(f"L2 traffic per launch: {l2:.4g} bytes (lts__t_sectors x 32 B) = {l2 / t_s / 1e9:.0f} GB/s")
        print()
        if a.traffic_json:
            t_i = h.index("gpu__time_duration.sum")
            with open(a.traffic_json, "w") as f:
                def pct(k):
                    return float(row[h.index(k)].replace(",", "")) if k in h and row[h.index(k)] else None

                json.dump({"kernel": row[name_i][:100], "dram_bytes_per_launch": rd + wr, "dram_read": rd,
                           "lts_throughput_pct": pct("lts__throughput.avg.pct_of_peak_sustained_elapsed"),
                           "l1tex_throughput_pct": pct("l1tex__throughput.avg.pct_of_peak_sustained_active"),
                           "issue_active_pct": pct("smsp__issue_active.avg.pct_of_peak_sustained_active"),
                           "l2_hit_rate_pct": pct("lts__t_sector_hit_rate.pct"),
                           "dram_write": wr, "l2_bytes_per_launch": l2, "report": a.rep,
                           "ncu_kernel_time": f"{row[t_i]} {units[t_i]}",
                           # the K1 sources this capture was taken of (bench.py flags stale captures)
                           "kernel_sha16": kernel_sha16()}, f, indent=1)
    if a.launches:
        rows = list(csv.reader(open(a.launches)))
        hi = [i for i, r in enumerate(rows) if "Kernel Name" in r][0]
        hh = rows[hi]
        idx = {n: i for i, n in enumerate(hh)}
        tot = collections.defaultdict(float)
        cnt = collections.Counter()
        mult = {"ns": 1e-6, "nsecond": 1e-6, "us": 1e-3, "usecond": 1e-3, "ms": 1.0, "msecond": 1.0, "s": 1e3}
        for r in rows[hi + 1:]:
            if len(r) < len(hh) or r[idx["Metric Name"]] != "gpu__time_duration.sum":
                continue
            k = r[idx["Kernel Name"]].split("(")[0][:70]
            tot[k] += float(r[idx["Metric Value"]].replace(",", "")) * mult.get(r[idx["Metric Unit"]], 1.0)
            cnt[k] += 1
        T = sum(tot.values()) or 1.0
        print("## launch list (ncu gpu__time_duration.sum, cold-cache, serialised)\n")
        print("| kernel | launches | total ms | share |\n|---|---|---|---|")
        for k, v in sorted(tot.items(), key=lambda x: -x[1]):
            print(f"| `{k}` | {cnt[k]} | {v:.3f} | {v / T * 100:.1f}% |")


if __name__ == "__main__":
    main()
