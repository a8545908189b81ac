#!/usr/bin/env python
"""Copy a measurement pass (scripts/gpu_profile_r1b.sh [tag], gpurun_out/<tag>/, default r1b) into profiles/:
bench lines, text outputs of the microbenchmarks / rates / traces, ncu summaries (JSON) of the
GEMV launches, the decode-loop microbenchmark and the persistent GEMV, the launch-list share table
and profiles/traffic.json (read by bench.py as roofline.traffic)."""
import csv
import io
import json
import os
import shutil
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
TAG = sys.argv[1] if len(sys.argv) > 1 else "r1b"                 # measurement pass label
SRC = os.path.join(ROOT, "gpurun_out", TAG)
DST = os.path.join(ROOT, "profiles")


def ncu_summary(rep, keys_extra=()):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    if len(rows) < 3:
        return {}
    head, units = rows[0], rows[1]
    scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "nsecond": 1e-3, "usecond": 1.0,
             "msecond": 1e3, "second": 1e6}
    res = {}
    for r in rows[2:]:
        d = dict(zip(head, r))
        u = dict(zip(head, units))
        name = d.get("Kernel Name", "?")
        rec = res.setdefault(name, {"launches": 0})
        rec["launches"] += 1

        def f(k):
            try:
                return float(d[k].replace(",", "")) * scale.get(u.get(k, ""), 1.0)
            except Exception:
                return None
        vals = {
            "duration_us": f("gpu__time_duration.sum") or 0.0,
            "dram_read_bytes": f("dram__bytes_read.sum"),
            "dram_write_bytes": f("dram__bytes_write.sum"),
            "issue_active_pct": f("smsp__issue_active.avg.pct_of_peak_sustained_active"),
            "alu_pipe_pct": f("sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_active"),
            "fma_pipe_pct": f("sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active"),
            "tensor_pipe_pct": f("sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active"),
            "registers": f("launch__registers_per_thread"),
            "grid": f("launch__grid_size"),
            "block": f("launch__block_size"),
        }
        for k, v in vals.items():
            if v is None:
                continue
            rec[k] = rec.get(k, 0.0) + v
        st = {}
        for k in head:
            if k.startswith("smsp__pcsamp_warps_issue_stalled_") and not k.endswith("_not_issued"):
                v = f(k)
                if v:
                    st[k.replace("smsp__pcsamp_warps_issue_stalled_", "")] = v
        tot = sum(st.values()) or 1.0
        rec.setdefault("_stalls", {})
        for k, v in st.items():
            rec["_stalls"][k] = rec["_stalls"].get(k, 0.0) + v / tot
    for name, rec in res.items():
        n = rec["launches"]
        for k in list(rec):
            if k not in ("launches", "_stalls"):
                rec[k] = rec[k] / n
        rec["stall_share_pct"] = {k: round(100 * v / n, 1) for k, v in sorted(rec.pop("_stalls").items(),
                                                                             key=lambda x: -x[1])[:8]}
        if rec.get("dram_read_bytes") is not None and rec.get("duration_us"):
            rec["dram_bytes_per_launch"] = rec["dram_read_bytes"] + (rec.get("dram_write_bytes") or 0)
            rec["dram_GBps"] = rec["dram_bytes_per_launch"] / (rec["duration_us"] * 1e-6) / 1e9
    return res


def launch_share(path):
    """Per-kernel share of the serialised ncu launch list (cold caches)."""
    with open(path) as f:
        lines = [ln for ln in f if ln.startswith('"')]
    rows = list(csv.reader(io.StringIO("".join(lines))))
    head = rows[0]
    ki, vi = head.index("Kernel Name"), head.index("Metric Value")
    tot = {}
    for r in rows[1:]:
        try:
            v = float(r[vi].replace(",", ""))
        except Exception:
            continue
        tot[r[ki]] = tot.get(r[ki], 0.0) + v
    s = sum(tot.values())
    return "\n".join(f"{100 * v / s:6.2f} %  {v / 1e3:10.1f} us  {k}" for k, v in sorted(tot.items(), key=lambda x: -x[1]))


def main():
    os.makedirs(DST, exist_ok=True)
    copies = {"bench.json": f"{TAG}_bench.json", "bench_reference.json": f"{TAG}_bench_reference.json",
              "c2_1mad.json": f"{TAG}_c2_1mad.json", "c4_70b_1gpu.json": f"{TAG}_c4_70b_1gpu.json",
              "c5_70b_hyb3_1gpu.json": f"{TAG}_c5_70b_hyb3_1gpu.json", "pipe_mix.txt": f"{TAG}_pipe_mix.txt",
              "decode_microbench.txt": f"{TAG}_decode_microbench.txt", "gridbar.txt": f"{TAG}_gridbar.txt",
              "gemv_rate.txt": f"{TAG}_gemv_rate.txt", "trace_fused_impl5.txt": f"{TAG}_trace_fused_impl5.txt",
              "trace_fused_impl6.txt": f"{TAG}_trace_fused_impl6.txt", "viterbi.txt": f"{TAG}_viterbi.txt",
              "gpu.txt": f"{TAG}_gpu.txt", "pytest_gpu.txt": f"{TAG}_pytest_gpu.txt", "smoke.txt": f"{TAG}_smoke.txt"}
    for a, b in copies.items():
        p = os.path.join(SRC, a)
        if os.path.exists(p):
            shutil.copy(p, os.path.join(DST, b))
    c3 = []
    for B in (1, 2, 4, 8, 16):
        p = os.path.join(SRC, f"c3_hyb4_b{B}.json")
        if os.path.exists(p):
            with open(p) as f:
                ln = [x for x in f.read().splitlines() if x.startswith("{")]
            if ln:
                c3.append(json.loads(ln[-1]))
    if c3:
        with open(os.path.join(DST, f"{TAG}_c3_hyb4_batch_sweep.json"), "w") as f:
            json.dump(c3, f, indent=1)
    for rep, out in (("prof_gemv", f"{TAG}_ncu_gemv.json"), ("prof_decode_loop", f"{TAG}_ncu_decode_loop.json"),
                     ("prof_gemv6", f"{TAG}_ncu_gemv6.json")):
        p = os.path.join(SRC, rep + ".ncu-rep")
        if os.path.exists(p):
            with open(os.path.join(DST, out), "w") as f:
                json.dump(ncu_summary(p), f, indent=1)
    lp = os.path.join(SRC, "launches.csv")
    if os.path.exists(lp):
        shutil.copy(lp, os.path.join(DST, f"{TAG}_launches.csv"))
        with open(os.path.join(DST, f"{TAG}_launches_summary.txt"), "w") as f:
            f.write(launch_share(lp) + "\n")
    # traffic.json for bench.py: mean DRAM bytes per GEMV launch of the 7B step
    gp = os.path.join(DST, f"{TAG}_ncu_gemv.json")
    if os.path.exists(gp):
        with open(gp) as f:
            g = json.load(f)
        tot_b, tot_n, names = 0.0, 0, []
        for k, v in g.items():
            if "dram_bytes_per_launch" in v:
                tot_b += v["dram_bytes_per_launch"] * v["launches"]
                tot_n += v["launches"]
                names.append(k)
        if tot_n:
            tp = os.path.join(DST, "traffic.json")
            t = json.load(open(tp)) if os.path.exists(tp) else {}
            # one block's GEMV launches (grouped q,k,v / gate,up count once): bytes per LAYER (7)
            t["llama2-7b/3inst/k2"] = {"dram_bytes_per_layer": tot_b / 7, "launches": tot_n, "kernels": names,
                                      "report": f"gpurun_out/{TAG}/prof_gemv.ncu-rep (profiles/{TAG}_ncu_gemv.json)"}
            with open(tp, "w") as f:
                json.dump(t, f, indent=1)
    print("ok")


if __name__ == "__main__":
    sys.exit(main())
