#!/usr/bin/env python
"""Summarise an `ncu --set full` report of bench.py's GEMV launches into profiles/.

usage: python scripts/ncu_traffic.py REPORT.ncu-rep KEY [OUT_JSON]

KEY is "<workload>/<code>/k<k>" (bench.py looks it up).  Writes, per kernel name, the mean over
the captured launches of duration, DRAM bytes read + written, achieved DRAM GB/s, issue-slot
utilisation and the top stall reasons, and records the GEMV entry under KEY in OUT_JSON
(default profiles/traffic.json).
"""
import csv
import io
import json
import os
import subprocess
import sys

UNITS = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "nsecond": 1e-9, "usecond": 1e-6, "msecond": 1e-3,
         "second": 1.0, "ns": 1e-9, "us": 1e-6, "ms": 1e-3, "s": 1.0, "%": 1.0, "": 1.0}


def raw(report):
    out = subprocess.run(["ncu", "-i", report, "--page", "raw", "--csv"], check=True, capture_output=True,
                         text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    head, units = rows[0], rows[1]
    recs = []
    for r in rows[2:]:
        d = {}
        for h, u, v in zip(head, units, r):
            try:
                d[h] = float(v.replace(",", "")) * UNITS.get(u, 1.0)
            except ValueError:
                d[h] = v
        recs.append(d)
    return recs


def summarise(recs):
    by = {}
    for d in recs:
        by.setdefault(d["Kernel Name"].split("(")[0], []).append(d)
    out = {}
    for name, ds in by.items():
        def mean(key):
            vals = [d[key] for d in ds if isinstance(d.get(key), float)]
            return sum(vals) / len(vals) if vals else None
        dur = mean("gpu__time_duration.sum")
        rd, wr = mean("dram__bytes_read.sum"), mean("dram__bytes_write.sum")
        s = {"launches": len(ds), "duration_us": dur * 1e6 if dur else None,
             "dram_bytes_per_launch": (rd or 0) + (wr or 0), "dram_read": rd, "dram_write": wr,
             "dram_GBps": ((rd or 0) + (wr or 0)) / dur / 1e9 if dur else None,
             "issue_active_pct": mean("sm__inst_issued.avg.pct_of_peak_sustained_active"),
             "warps_active_pct": mean("sm__warps_active.avg.pct_of_peak_sustained_active"),
             "registers": mean("launch__registers_per_thread"),
             "grid": ds[0].get("launch__grid_size"), "block": ds[0].get("launch__block_size")}
        stalls = {}
        for key in ds[0]:
            if key.startswith("smsp__average_warps_issue_stalled_") and key.endswith("_per_issue_active.ratio"):
                v = mean(key)
                if v:
                    stalls[key[len("smsp__average_warps_issue_stalled_"):-len("_per_issue_active.ratio")]] = v
        s["stalls_per_issue"] = dict(sorted(stalls.items(), key=lambda kv: -kv[1])[:8])
        out[name] = s
    return out


def main():
    report, key = sys.argv[1], sys.argv[2]
    path = sys.argv[3] if len(sys.argv) > 3 else os.path.join(os.path.dirname(__file__), "..", "profiles",
                                                              "traffic.json")
    recs = raw(report)
    summ = summarise(recs)
    # all GEMV launches of the capture together (the bench's per-launch average runs over the
    # step's mix of kernels)
    g = [d for d in recs if "gemv" in d["Kernel Name"]]
    if g:
        tot = sum(d.get("dram__bytes_read.sum", 0.0) + d.get("dram__bytes_write.sum", 0.0) for d in g)
        dur = sum(d["gpu__time_duration.sum"] for d in g)
        summ["all_gemv"] = {"launches": len(g), "dram_bytes_per_launch": tot / len(g),
                            "duration_us": dur / len(g) * 1e6, "dram_GBps": tot / dur / 1e9,
                            "kernels": sorted(set(d["Kernel Name"].split("(")[0] for d in g))}
    print(json.dumps(summ, indent=1))
    gemv = [summ["all_gemv"]] if g else []
    if gemv:
        try:
            with open(path) as f:
                db = json.load(f)
        except Exception:
            db = {}
        db[key] = dict(gemv[0], report=os.path.basename(report))
        with open(path, "w") as f:
            json.dump(db, f, indent=1, sort_keys=True)


if __name__ == "__main__":
    main()
