#!/usr/bin/env python
"""Summarise an ncu launch list (CSV from `ncu --metrics gpu__time_duration.sum,
dram__bytes_read.sum,dram__bytes_write.sum --csv`) of a bench.py run.

    python tools/launch_list.py LAUNCHES.csv WORKLOAD OUT.txt [--traffic profiles/ncu_traffic.json]

Writes one line per launch plus a per-kernel-kind table (launches after the
synthetic fill; mean time, mean DRAM bytes, share of the step) and, with
--traffic, records the mean DRAM bytes per launch of each kind under
WORKLOAD in the traffic JSON that bench.py reports as roofline.traffic.
Times are cold-cache and serialised (ncu replay): compare SHARES, not ms.
"""
import argparse
import csv
import json
import os
import re
from collections import defaultdict

KINDS = [("segment_kernel", "segment"), ("simt_shrink", "simt_shrink"), ("simt_expand", "simt_expand"),
         ("tc_shrink", "tc05_shrink"), ("tc_vreduce", "tc05_vreduce"), ("tc_expand", "tc05_expand"),
         ("bucket_kernel", "shard_bucket"), ("gather_", "shard_gather"), ("scatter_add", "shard_scatter_add")]
SCALE = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "KB": 1e3, "MB": 1e6, "GB": 1e9}
TSCALE = {"nsecond": 1e-9, "ns": 1e-9, "usecond": 1e-6, "us": 1e-6, "msecond": 1e-3, "ms": 1e-3}


def kind_of(name):
    for pat, k in KINDS:
        if pat in name:
            return k
    return None


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("csv")
    ap.add_argument("workload")
    ap.add_argument("out")
    ap.add_argument("--traffic", default=None)
    a = ap.parse_args()
    text = open(a.csv).read()
    lines = [l for l in text.splitlines() if l.startswith('"')]
    rows = list(csv.reader(lines))
    hdr = rows[0]
    c = {h: i for i, h in enumerate(hdr)}
    launches = {}
    for r in rows[1:]:
        if len(r) != len(hdr) or not r[c["ID"]].isdigit():
            continue
        lid = int(r[c["ID"]])
        d = launches.setdefault(lid, {"name": r[c["Kernel Name"]]})
        v = float(r[c["Metric Value"]].replace(",", ""))
        u = r[c["Metric Unit"]]
        m = r[c["Metric Name"]]
        if m == "gpu__time_duration.sum":
            d["t"] = v * TSCALE.get(u, 1e-9)
        elif m == "dram__bytes_read.sum":
            d["rd"] = v * SCALE.get(u, 1)
        elif m == "dram__bytes_write.sum":
            d["wr"] = v * SCALE.get(u, 1)
    per = defaultdict(lambda: [0, 0.0, 0.0])
    out = [f"# ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none",
           f"# python bench.py --workload {a.workload} (cold-cache serialised replay: compare shares, not ms)"]
    for lid in sorted(launches):
        d = launches[lid]
        k = kind_of(d["name"])
        out.append(f"{lid:5d} {d['name'][:60]:60s} {d.get('t', 0) * 1e6:10.2f} us  read {d.get('rd', 0) / 1e6:10.2f} MB"
                   f"  write {d.get('wr', 0) / 1e6:9.2f} MB")
        if k:
            p = per[k]
            p[0] += 1
            p[1] += d.get("t", 0)
            p[2] += d.get("rd", 0) + d.get("wr", 0)
    tot = sum(p[1] for p in per.values()) or 1
    out.append("")
    out.append(f"{'kind':20s} {'launches':>8s} {'mean us':>10s} {'mean MB':>10s} {'GB/s':>8s} {'share':>6s}")
    for k, (n, t, b) in sorted(per.items(), key=lambda x: -x[1][1]):
        out.append(f"{k:20s} {n:8d} {t / n * 1e6:10.2f} {b / n / 1e6:10.2f} {b / t / 1e9:8.0f} {100 * t / tot:5.1f}%")
    open(a.out, "w").write("\n".join(out) + "\n")
    print("\n".join(out[-len(per) - 1:]))
    if a.traffic:
        tj = json.load(open(a.traffic)) if os.path.exists(a.traffic) else {}
        tj[a.workload] = {k: b / n for k, (n, t, b) in per.items()}
        tj["_source"] = "tools/launch_list.py over profiles/*launches*.txt (ncu dram__bytes_read.sum + " \
                        "dram__bytes_write.sum, mean per launch)"
        json.dump(tj, open(a.traffic, "w"), indent=1)


if __name__ == "__main__":
    main()
