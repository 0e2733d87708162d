#!/usr/bin/env python
"""Summarise an ncu report: per kernel time, DRAM bytes/throughput, issue
activity, top stall reasons and (optionally) the hottest SASS lines.

    python tools/ncu_summary.py REPORT.ncu-rep [--source REGEX] [--top N]
"""
import argparse
import csv
import io
import subprocess
import sys


def ncu_csv(args):
    out = subprocess.run(["ncu"] + args + ["--csv"], capture_output=True, text=True).stdout
    return list(csv.reader(io.StringIO(out)))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("report")
    ap.add_argument("--source", default=None)
    ap.add_argument("--top", type=int, default=20)
    a = ap.parse_args()
    rows = ncu_csv(["-i", a.report, "--page", "raw"])
    hdr, units = rows[0], rows[1]
    col = {h: i for i, h in enumerate(hdr)}

    def g(r, k):
        i = col.get(k)
        return r[i] if i is not None else ""

    for r in rows[2:]:
        name = g(r, "Kernel Name")
        t = float(g(r, "gpu__time_duration.sum") or 0)
        tu = units[col["gpu__time_duration.sum"]]
        rd = float(g(r, "dram__bytes_read.sum") or 0)
        wr = float(g(r, "dram__bytes_write.sum") or 0)
        ru, wu = units[col["dram__bytes_read.sum"]], units[col["dram__bytes_write.sum"]]
        scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}
        tscale = {"ns": 1e-9, "us": 1e-6, "usecond": 1e-6, "ms": 1e-3, "msecond": 1e-3, "nsecond": 1e-9}
        secs = t * tscale.get(tu, 1e-3)
        byts = rd * scale.get(ru, 1) + wr * scale.get(wu, 1)
        print(f"{name[:70]}")
        print(f"   time {t:.4f} {tu}   dram read {rd:.3f} {ru} write {wr:.3f} {wu}   -> {byts / secs / 1e9:.0f} GB/s")
        for k in ["dram__throughput.avg.pct_of_peak_sustained_elapsed", "smsp__issue_active.avg.pct_of_peak_sustained_active",
                  "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active", "launch__registers_per_thread",
                  "launch__occupancy_limit_registers", "sm__warps_active.avg.pct_of_peak_sustained_active",
                  "lts__t_sector_hit_rate.pct"]:
            if k in col:
                print(f"   {k:70s} {g(r, k)}")
        st = {}
        for h, i in col.items():
            if h.startswith("smsp__pcsamp_warps_issue_stalled_") and not h.endswith("not_issued"):
                try:
                    st[h.replace("smsp__pcsamp_warps_issue_stalled_", "")] = float(r[i])
                except ValueError:
                    pass
        tot = sum(st.values()) or 1
        print("   stalls: " + ", ".join(f"{k} {100 * v / tot:.0f}%" for k, v in sorted(st.items(), key=lambda x: -x[1])[:7]))
    if a.source:
        src = ncu_csv(["-i", a.report, "--page", "source", "-k", "regex:" + a.source])
        h = src[1]
        data = [r for r in src[2:] if len(r) == len(h)]
        si = h.index("Warp Stall Sampling (All Samples)")
        seen, ded = set(), []
        for r in data:
            if r[0] not in seen:
                seen.add(r[0])
                ded.append(r)
        v = lambda r: int(r[si]) if r[si].strip().isdigit() else 0
        tot = sum(v(r) for r in ded) or 1
        print(f"hot SASS ({a.source}), {tot} samples:")
        for r in sorted(ded, key=lambda r: -v(r))[:a.top]:
            print(f"   {100 * v(r) / tot:5.1f}%  {r[1][:110]}")


if __name__ == "__main__":
    main()
