#!/usr/bin/env python
"""QTIP fused trellis-decode GEMV benchmark (BASELINE.json metric: compressed-byte HBM GB/s vs
peak; us/layer at batch 1).

Step (default workload `llama2-7b`, BASELINE configs[1]): one batch-1 decode token through the
linear layers of all 32 Llama-2-7B decoder blocks -- q, k, v, o (4096x4096), gate, up
(11008x4096), down (4096x11008) -- each layer = RHT-in -> fused decode-GEMV -> RHT-out, k=2 3INST,
L=16, V=1, T=256 tail-biting, every layer its own weights (1.62 GB of packed stream > 126 MB L2,
so no layer is L2-resident when it is read again next step).  Within a block the model's data
dependencies hold: q, k, v (same input) run concurrently, then o, then gate and up concurrently,
then down (fork/join streams inside the CUDA graph); config.step_serial_ms is the same step with
every layer strictly after the previous one.  value = compressed bytes / step time (GB/s), whole
job.  With torchrun (N>1) every layer is row-sharded across ranks and the
y~ shards are all-gathered over NCCL before the replicated RHT-out (strong scaling).

`--impl reference` times the CPU oracle (the tier's reference arm) on a bounded sample.
"""
import argparse
import json
import os
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

import synth  # noqa: E402

WORKLOADS = {
    # name: (blocks, [(m, n) per linear in a block], default code, default k)
    "llama2-7b": (32, [(4096, 4096)] * 4 + [(11008, 4096)] * 2 + [(4096, 11008)], "3inst", 2),
    "llama2-70b": (80, [(8192, 8192), (1024, 8192), (1024, 8192), (8192, 8192), (28672, 8192), (28672, 8192),
                        (8192, 28672)], "hyb", 3),
    "c4-70b": (8, [(8192, 28672), (28672, 8192)], "3inst", 2),
    # the 7B block with q,k,v and gate,up stacked into one matrix each (one RHT over the stacked
    # output): the same weight bytes in 4 layers per block
    "llama2-7b-stacked": (32, [(12288, 4096), (4096, 4096), (22016, 4096), (4096, 11008)], "3inst", 2),
}
# Data dependencies inside a block (the model's): q, k, v read the same normalised input, as do
# gate and up, so each group runs concurrently (fork/join streams inside the graph); the groups
# themselves are sequential (o needs attention over q, k, v; down needs silu(gate) * up).
GROUPS = {
    "llama2-7b": [[0, 1, 2], [3], [4, 5], [6]],
    "llama2-70b": [[0, 1, 2], [3], [4, 5], [6]],
    "c4-70b": [[0], [1]],
    "llama2-7b-stacked": [[0], [1], [2], [3]],
}


# The step is a chain (the model's data flow): the first group of block 0 reads the external x; every
# later group reads the output of one layer of the previous group -- o reads q's output (a stand-in
# for attention), gate and up read o's, down reads gate's (a stand-in for silu(gate) * up), the next
# block's q, k, v read down's.  CHAIN_SRC[workload][g] = index within group g-1 of that layer.
CHAIN_SRC = {
    "llama2-7b": [0, 0, 0, 0],
    "llama2-70b": [0, 0, 0, 0],
    "c4-70b": [0, 0],
}
# code variance over the 2^16 states (R9): scale = 1 / sqrt(n var) keeps |y| ~ |x| along the chain
CODE_VAR = {"3inst": 1.547, "1mad": 1.0, "hyb": 1.0}


def peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            d = json.load(f)
        return float(d["hbm_gbs"]), "measured"
    except Exception:
        return 6650.0, "fallback"


def traffic(workload, code, k, impl):
    """DRAM bytes (read + write) per layer of the step's GEMV launches from the committed
    `ncu --set full` capture of one block (profiles/traffic.json, written by
    scripts/summarize_r1b.py), or None if not captured."""
    try:
        with open(os.path.join(ROOT, "profiles", "traffic.json")) as f:
            d = json.load(f)
        return d[f"{workload}/{code}/k{k}"]["dram_bytes_per_layer"]
    except Exception:
        return None


# ---------------------------------------------------------------------------- clocks
class ClockSampler:
    FIELDS = "clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown," \
             "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap"

    def __init__(self, index):
        self.index = index
        self.proc = None
        self.lines = []

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.FIELDS}",
                                          "--format=csv,noheader,nounits", "-lms", "100"],
                                         stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except Exception:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def __exit__(self, *a):
        if self.proc is not None:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except Exception:
                self.proc.kill()

    def summary(self):
        sm, mx, reasons = [], [], set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in self.lines:
            parts = [p.strip() for p in ln.split(",")]
            if len(parts) < 6:
                continue
            try:
                sm.append(float(parts[0]))
                mx.append(float(parts[1]))
            except ValueError:
                continue
            for nm, v in zip(names, parts[2:6]):
                if v.lower().startswith("active"):
                    reasons.add(nm)
        if not sm:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"]}
        return {"sm_mhz": float(np.median(sm)), "sm_max_mhz": float(max(mx)), "reasons": sorted(reasons),
                "samples": len(sm)}


# ---------------------------------------------------------------------------- CPU oracle
def oracle_sample(m=2048, n=4096, code="3inst", k=2, reps=1):
    """Plain oracle (single thread): decode + float64 RHT-in / GEMV / RHT-out of one m x n layer."""
    from threadpoolctl import threadpool_limits
    from oracle import gemv
    tiles = synth.random_tiles(m, n, k, seed=1000)
    lut = synth.gaussian_lut(9) if code == "hyb" else None
    x = synth.random_x(1, n).astype(np.float64)
    sm, sn = synth.random_sign_bytes(m, 3001), synth.random_sign_bytes(n, 3000)
    p = gemv.Params(k=k, V=2 if code == "hyb" else 1, code=code, lut=lut)
    times = []
    with threadpool_limits(1):
        for _ in range(reps):
            t0 = time.perf_counter()
            W = gemv.dense_decode(tiles, p)
            gemv.matvec(W, x, sn, sm, scale=1.0)
            times.append(time.perf_counter() - t0)
    nbytes = m * n * k / 8
    return nbytes, times


def _oracle_rows_worker(job):
    """One process of the all-cores oracle: decode a block of tile rows and form its rows of W~ x~."""
    from threadpoolctl import threadpool_limits
    from oracle import gemv
    m, n, k, code, I0, I1, xt = job
    tiles = synth.random_tiles(m, n, k, seed=1000)[I0:I1]
    lut = synth.gaussian_lut(9) if code == "hyb" else None
    p = gemv.Params(k=k, V=2 if code == "hyb" else 1, code=code, lut=lut)
    with threadpool_limits(1):
        return I0, xt @ gemv.dense_decode(tiles, p).T


def oracle_sample_all_cores(m=2048, n=4096, code="3inst", k=2, procs=None):
    """The same oracle computation split over all host cores (a process pool over tile-row blocks;
    the RHTs stay on the parent).  Returns (bytes, seconds, processes)."""
    import multiprocessing as mproc
    from oracle import rht
    procs = procs or os.cpu_count() or 1
    x = synth.random_x(1, n).astype(np.float64)
    sm, sn = synth.random_sign_bytes(m, 3001), synth.random_sign_bytes(n, 3000)
    mt = m // 16
    blocks = [(i * mt // procs, (i + 1) * mt // procs) for i in range(procs)]
    with mproc.get_context("spawn").Pool(procs) as pool:
        pool.map(_oracle_rows_worker, [(256, 256, k, code, 0, 16, np.zeros((1, 256)))] * procs)   # warm
        t0 = time.perf_counter()
        xt = rht.rht_forward(x, sn, n)
        yt = np.zeros((1, m))
        for I0, part in pool.map(_oracle_rows_worker, [(m, n, k, code, a, b, xt) for a, b in blocks if b > a]):
            yt[:, 16 * I0:16 * I0 + part.shape[1]] = part
        rht.rht_inverse(yt, sm, m)
        dt = time.perf_counter() - t0
    return m * n * k / 8, dt, procs


def cpu_model():
    try:
        with open("/proc/cpuinfo") as f:
            for line in f:
                if line.startswith("model name"):
                    return line.split(":", 1)[1].strip()
    except OSError:
        pass
    return "unknown"


def cpu_baseline(code, k):
    """The oracle timed on this host: single thread (the reference arm's setting) and all cores, on a
    2048 x 4096 sample of the workload's code; microseconds per layer extrapolated from the
    per-weight time (decode dominates; the RHTs are < 3 %) for the C1-C3 shapes."""
    nbytes, times = oracle_sample(2048, 4096, code, k, reps=2)
    t1 = min(times)
    nb_all, t_all, procs = oracle_sample_all_cores(2048, 4096, code, k)
    per_w1, per_wN = t1 / (2048 * 4096), t_all / (2048 * 4096)
    shapes = {"256x256": 256 * 256, "4096x4096": 4096 * 4096, "11008x4096": 11008 * 4096, "4096x11008": 4096 * 11008}
    return {"value": round(nbytes / t1 / 1e9, 5), "unit": "GB/s", "cores": 1, "kind": "oracle",
            "sample": f"2 x one 2048x4096 {code} k={k} layer (decode + float64 RHT-in/GEMV/RHT-out), single thread "
                      f"(best of 2); all-cores: the same layer split over a {procs}-process pool",
            "cpu_model": cpu_model(), "host_cores": os.cpu_count(),
            "all_cores": {"value": round(nb_all / t_all / 1e9, 5), "unit": "GB/s", "cores": procs},
            "us_per_layer_1_core": {s: round(per_w1 * w * 1e6, 0) for s, w in shapes.items()},
            "us_per_layer_all_cores": {s: round(per_wN * w * 1e6, 0) for s, w in shapes.items()}}


def run_reference(args):
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    wl = WORKLOADS[args.workload]
    code = args.code or wl[2]
    k = args.k or wl[3]
    m, n = 2048, 4096
    oracle_sample(256, 256, code, k, reps=1)                       # import / table warm-up
    for _ in range(args.warmup):
        oracle_sample(m, n, code, k, reps=1)
    nbytes, times = oracle_sample(m, n, code, k, reps=args.steps)
    tot = sum(times)
    value = nbytes * args.steps / tot / 1e9
    sample = f"one {m}x{n} {code} k={k} layer per step (decode + float64 RHT-in/GEMV/RHT-out), single thread"
    line = {"metric": "fused trellis-decode GEMV: compressed-byte HBM GB/s vs peak; us/layer batch=1",
            "value": value, "unit": "GB/s", "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": 1e3 * tot / args.steps, "higher_is_better": True, "scaling": "weak",
            "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": {"workload": args.workload, "code": code, "k": k, "batch": 1, "sample": sample},
            "impl": "reference",
            "cpu_baseline": {"value": value, "unit": "GB/s", "cores": 1, "kind": "oracle", "sample": sample},
            "e2e": {"value": value, "unit": "GB/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


# ---------------------------------------------------------------------------- GPU arm
def run_ours(args):
    import torch
    import torch.distributed as dist

    from paper_2406_11235_b200 import qtip
    from paper_2406_11235_b200.layer import QTIPLinear, forward_group
    from paper_2406_11235_b200.sharded import ShardedQTIPLinear

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world != args.gpus:
        raise SystemExit(f"bench.py: --gpus {args.gpus} but WORLD_SIZE={world} (launch N ranks with torchrun, or let "
                         "bench.py relaunch itself)")
    if local >= torch.cuda.device_count():
        raise SystemExit(f"bench.py: rank {rank} needs GPU {local} but only {torch.cuda.device_count()} visible")
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if world > 1:
        # communicator lines (nRanks, NVLS / P2P transport) in the log; the JSON line stays last on stdout
        os.environ.setdefault("NCCL_DEBUG", "INFO")
        os.environ.setdefault("NCCL_DEBUG_SUBSYS", "INIT")
        dist.init_process_group("nccl", device_id=dev)
    qtip.load()
    qtip.set_matvec_impl(args.matvec_impl)
    if os.environ.get("QTIP_L2_PREFETCH") is not None:       # ablation: MiB of weights the RHT-in prefetches (0 = off)
        qtip.load().qtip_internal_set_knob(4, int(os.environ["QTIP_L2_PREFETCH"]))

    nblocks, shapes, dcode, dk = WORKLOADS[args.workload]
    if args.blocks:
        nblocks = args.blocks
    code = args.code or dcode
    k = args.k or dk
    B = args.batch
    lut = synth.gaussian_lut(9) if code == "hyb" else None

    # one prototype per distinct shape, copied device-to-device into every layer instance
    protos = {}
    for si, (m, n) in enumerate(sorted(set(shapes))):
        tiles = synth.random_tiles(m, n, k, seed=1000 + si)
        sm, sn = synth.random_sign_bytes(m, 3001 + si), synth.random_sign_bytes(n, 3000 + si)
        if world == 1:
            lay = QTIPLinear(m, n, code=code, k=k, device=dev).load_tiles(tiles, sm, sn, scale=1.0 / np.sqrt(n * CODE_VAR[code]),
                                                                          lut=lut)
        else:
            lay = ShardedQTIPLinear(m, n, rank, world, code=code, k=k, device=dev).load_tiles(tiles, sm, sn, lut=lut)
        protos[(m, n)] = lay
        del tiles
    layers = []
    for b in range(nblocks):
        for (m, n) in shapes:
            pr = protos[(m, n)]
            if world == 1:
                lay = QTIPLinear(m, n, code=code, k=k, device=dev)
                lay.packed.copy_(pr.packed)
                lay.sign_m.copy_(pr.sign_m)
                lay.sign_n.copy_(pr.sign_n)
                lay.lut, lay.scale = pr.lut, pr.scale
            else:
                lay = ShardedQTIPLinear(m, n, rank, world, code=code, k=k, device=dev)
                lay.local.packed.copy_(pr.local.packed)
                lay.local.sign_n.copy_(pr.local.sign_n)
                lay.local.lut, lay.local.scale = pr.local.lut, pr.local.scale
                lay.sign_m.copy_(pr.sign_m)
            layers.append(lay)
    del protos
    torch.cuda.synchronize()

    ns = sorted(set(n for _, n in shapes))
    xs = {n: torch.from_numpy(synth.random_x(B, n, seed=2000 + n)).to(dev) for n in ns}
    outs = [torch.empty((B, lay.m), dtype=torch.float32, device=dev) for lay in layers]
    step_bytes = sum(m * n * k // 8 for (m, n) in shapes) * nblocks


    nl_blk = len(shapes)
    groups = GROUPS[args.workload]
    side = [torch.cuda.Stream(device=dev) for _ in range(max(len(g) for g in groups) - 1)]
    chained = args.workload in CHAIN_SRC and world == 1
    src_of = {}                                       # layer index -> layer index whose output it reads
    if chained:
        for blk in range(nblocks):
            for gi, grp in enumerate(groups):
                if blk == 0 and gi == 0:
                    continue
                pg = groups[gi - 1] if gi > 0 else groups[-1]
                pb = blk if gi > 0 else blk - 1
                for i in grp:
                    src_of[blk * nl_blk + i] = pb * nl_blk + pg[CHAIN_SRC[args.workload][gi]]

    def input_of(i):
        return outs[src_of[i]] if i in src_of else xs[layers[i].n]

    def run_layer(i):
        lay, o = layers[i], outs[i]
        if world == 1:
            lay.forward(input_of(i), out=o)
        else:
            o.copy_(lay.forward(xs[lay.n]))

    def step(serial=False):
        nl = len(shapes)
        for blk in range(nblocks):
            for grp in groups:
                if not serial and len(grp) > 1 and args.grouping == "launch" and world == 1:
                    # same-shape layers on one input: one grouped call (qtip_matvec_group) per shape;
                    # differently shaped members (70B: q vs k, v) run concurrently on side streams
                    by_shape = {}
                    for i in grp:
                        by_shape.setdefault(shapes[i], []).append(blk * nl + i)
                    parts = list(by_shape.values())

                    def run_part(idx):
                        if len(idx) == 1:
                            run_layer(idx[0])
                        else:
                            forward_group([layers[i] for i in idx], input_of(idx[0]), outs=[outs[i] for i in idx])
                    if len(parts) == 1:
                        run_part(parts[0])
                        continue
                    cur = torch.cuda.current_stream()
                    for si in range(len(parts) - 1):
                        side[si].wait_stream(cur)
                    run_part(parts[0])
                    for si, idx in enumerate(parts[1:]):
                        with torch.cuda.stream(side[si]):
                            run_part(idx)
                    for si in range(len(parts) - 1):
                        cur.wait_stream(side[si])
                    continue
                if serial or len(grp) == 1 or args.grouping == "serial":
                    for i in grp:
                        run_layer(blk * nl + i)
                    continue
                cur = torch.cuda.current_stream()
                for si in range(len(grp) - 1):                  # fork after the previous group
                    side[si].wait_stream(cur)
                run_layer(blk * nl + grp[0])
                for si, i in enumerate(grp[1:]):
                    with torch.cuda.stream(side[si]):
                        run_layer(blk * nl + i)
                for si in range(len(grp) - 1):                  # join
                    cur.wait_stream(side[si])

    # eager warm-up (Hadamard tables, workspaces, NCCL communicators), then capture one step
    for _ in range(2):
        step()
    torch.cuda.synchronize()
    c0 = qtip.launch_count()
    g = torch.cuda.CUDAGraph()
    s = torch.cuda.Stream()
    s.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(s):
        with torch.cuda.graph(g, stream=s):
            step()
    torch.cuda.current_stream().wait_stream(s)
    launches_per_step = qtip.launch_count() - c0
    torch.cuda.synchronize()

    def barrier():
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()

    def max_over_ranks(v):
        if world == 1:
            return v
        t = torch.tensor([v], dtype=torch.float64, device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return float(t.item())

    for _ in range(max(3, args.warmup)):
        g.replay()
    barrier()
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with ClockSampler(local) as clk:
        ev0.record()
        for _ in range(args.steps):
            g.replay()
        ev1.record()
        torch.cuda.synchronize()
    barrier()
    ms = max_over_ranks(ev0.elapsed_time(ev1) / args.steps)
    value = step_bytes / (ms * 1e-3) / 1e9

    # the same step with every layer strictly after the previous one (no group concurrency)
    gs = torch.cuda.CUDAGraph()
    with torch.cuda.stream(s):
        with torch.cuda.graph(gs, stream=s):
            step(serial=True)
    torch.cuda.current_stream().wait_stream(s)
    for _ in range(3):
        gs.replay()
    barrier()
    es0, es1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    es0.record()
    for _ in range(args.steps):
        gs.replay()
    es1.record()
    torch.cuda.synchronize()
    ms_serial = max_over_ranks(es0.elapsed_time(es1) / args.steps)
    del gs

    # ---- per-shape layer latency (graph of one layer, replayed) for us/layer reporting
    per_layer = {}
    for (m, n) in sorted(set(shapes)):
        idx = [i for i, l in enumerate(layers) if (l.m, l.n) == (m, n)]
        gl = torch.cuda.CUDAGraph()
        with torch.cuda.stream(s):
            with torch.cuda.graph(gl, stream=s):
                for i in idx:
                    if world == 1:
                        layers[i].forward(xs[n], out=outs[i])
                    else:
                        outs[i].copy_(layers[i].forward(xs[n]))
        torch.cuda.current_stream().wait_stream(s)
        for _ in range(3):
            gl.replay()
        barrier()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(max(1, args.steps // 2)):
            gl.replay()
        e1.record()
        torch.cuda.synchronize()
        us = max_over_ranks(1e3 * e0.elapsed_time(e1) / (max(1, args.steps // 2) * len(idx)))
        per_layer[f"{m}x{n}"] = {"us_per_layer": round(us, 3),
                                 "GBps": round(m * n * k / 8 / (us * 1e-6) / 1e9, 1)}
        if world == 1:
            # spread over single-layer replays (each bracketed by its own events, which add a few us of
            # event overhead: a distribution, not the step's per-layer time) and one cold call (L2
            # flushed by a 256 MB write, eager launches)
            l0 = layers[idx[0]]
            g1 = torch.cuda.CUDAGraph()
            with torch.cuda.stream(s):
                with torch.cuda.graph(g1, stream=s):
                    l0.forward(xs[n], out=outs[idx[0]])
            torch.cuda.current_stream().wait_stream(s)
            g1.replay()
            single = []
            for _ in range(20):
                a0, a1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                a0.record()
                g1.replay()
                a1.record()
                torch.cuda.synchronize()
                single.append(1e3 * a0.elapsed_time(a1))
            flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)
            flush.fill_(1)
            a0, a1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a0.record()
            l0.forward(xs[n], out=outs[idx[0]])
            a1.record()
            torch.cuda.synchronize()
            del flush, g1
            per_layer[f"{m}x{n}"].update({"single_replay_us_p10_p50_p90": [round(float(v), 2) for v in np.percentile(single, [10, 50, 90])],
                                          "cold_call_us": round(1e3 * a0.elapsed_time(a1), 2)})

    # ---- dominant kernel (fused decode-GEMV): the step's GEMV launches alone, back to back in a
    #      graph (each layer's x~ is already in its workspace: QTIP_XT_READY skips the RHT-in;
    #      RHT-out off; PDL on), timed with CUDA events around the replays
    locs = [(lay if world == 1 else lay.local) for lay in layers]
    gouts = [torch.empty((B, t.m), dtype=torch.float32, device=dev) for t in locs]
    gflags = qtip.QTIP_RHT_IN | qtip.QTIP_XT_READY

    def gemv_launches():
        # the step's decode-GEMV launches in step order (grouped layers as one grouped launch)
        nl = len(shapes)
        for blk in range(nblocks):
            for grp in groups:
                parts = {}
                for i in grp:
                    parts.setdefault(shapes[i], []).append(blk * nl + i)
                for idx in parts.values():
                    if len(idx) > 1 and args.grouping == "launch" and world == 1:
                        forward_group([locs[i] for i in idx], xs[locs[idx[0]].n], outs=[gouts[i] for i in idx],
                                      flags=gflags)
                    else:
                        for i in idx:
                            locs[i].forward(xs[locs[i].n], out=gouts[i], flags=gflags)

    gk = torch.cuda.CUDAGraph()
    with torch.cuda.stream(s):
        step()                                                  # x~ of every layer in its workspace
        gemv_launches()                                         # eager pass
        with torch.cuda.graph(gk, stream=s):
            gemv_launches()
    torch.cuda.current_stream().wait_stream(s)
    for _ in range(3):
        gk.replay()
    barrier()
    prof_steps = max(1, args.steps)
    g0, g1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    g0.record()
    for _ in range(prof_steps):
        gk.replay()
    g1.record()
    torch.cuda.synchronize()
    gemv_ms = max_over_ranks(g0.elapsed_time(g1))
    gemv_bytes = prof_steps * sum(t.m * t.n * k // 8 for t in locs)
    gemv_gbs = gemv_bytes / (gemv_ms * 1e-3) / 1e9
    del gk, gouts
    peak, peak_kind = peaks()

    # ---- end to end through the public API: pinned H2D of x, the step, D2H of the last output
    xh = {n: torch.from_numpy(synth.random_x(B, n, seed=2000 + n)).pin_memory() for n in ns}
    yh = torch.empty_like(outs[-1], device="cpu").pin_memory()
    ge = torch.cuda.CUDAGraph()
    with torch.cuda.stream(s):
        with torch.cuda.graph(ge, stream=s):
            for n in ns:
                xs[n].copy_(xh[n], non_blocking=True)
            step()
            yh.copy_(outs[-1], non_blocking=True)
    torch.cuda.current_stream().wait_stream(s)
    for _ in range(3):
        ge.replay()
    barrier()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(args.steps):
        ge.replay()
    e1.record()
    torch.cuda.synchronize()
    e2e_ms = max_over_ranks(e0.elapsed_time(e1) / args.steps)
    h2d = sum(x.numel() * 4 for x in xh.values())
    d2h = yh.numel() * 4
    layers_path = {"ms_per_step": round(ms, 5), "GBps": round(value, 2), "e2e_ms_per_step": round(e2e_ms, 5),
                   "step_serial_ms": round(ms_serial, 5), "gemv_only_GBps": round(gemv_gbs, 1),
                   "launches_per_step": launches_per_step}

    # ---- the chain kernel (impl 8, qtip_chain_run): the whole step -- every layer, its RHT-in, GEMV
    #      and RHT-out, and the stage hand-offs -- as ONE persistent launch
    chain_res = None
    if args.path == "chain" and chained and B <= 16:
        from paper_2406_11235_b200.layer import QTIPChain
        cstages = []
        for blk in range(nblocks):
            for gi, grp in enumerate(groups):
                cstages.append(([layers[blk * nl_blk + i] for i in grp], CHAIN_SRC[args.workload][gi]))
        chain = QTIPChain(cstages, B=B)
        x0 = xs[layers[0].n]
        chain(x0)
        torch.cuda.synchronize()
        c0 = qtip.launch_count()
        gch = torch.cuda.CUDAGraph()
        with torch.cuda.stream(s):
            with torch.cuda.graph(gch, stream=s):
                chain(x0)
        torch.cuda.current_stream().wait_stream(s)
        launches_chain = qtip.launch_count() - c0
        for _ in range(max(3, args.warmup)):
            gch.replay()
        barrier()
        h0, h1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        with ClockSampler(local) as clk:
            h0.record()
            for _ in range(args.steps):
                gch.replay()
            h1.record()
            torch.cuda.synchronize()
        ms_chain = max_over_ranks(h0.elapsed_time(h1) / args.steps)
        # end to end: pinned H2D of x, the chain, D2H of the last layer's output, all in the timed graph
        xh0 = torch.from_numpy(synth.random_x(B, layers[0].n, seed=2000 + layers[0].n)).pin_memory()
        yl = chain.outs[-1][-1]
        yh0 = torch.empty(tuple(yl.shape), dtype=torch.float32).pin_memory()
        gce = torch.cuda.CUDAGraph()
        with torch.cuda.stream(s):
            with torch.cuda.graph(gce, stream=s):
                x0.copy_(xh0, non_blocking=True)
                chain(x0)
                yh0.copy_(yl, non_blocking=True)
        torch.cuda.current_stream().wait_stream(s)
        for _ in range(3):
            gce.replay()
        barrier()
        f0, f1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        f0.record()
        for _ in range(args.steps):
            gce.replay()
        f1.record()
        torch.cuda.synchronize()
        e2e_chain = max_over_ranks(f0.elapsed_time(f1) / args.steps)
        chain_res = {"ms": ms_chain, "e2e_ms": e2e_chain, "h2d": xh0.numel() * 4, "d2h": yh0.numel() * 4,
                     "launches": launches_chain, "stages": len(cstages)}
        del gch, gce
        chain.close()

    # ---- C4 (BASELINE configs[3]): the 70B layers 8192x28672 and 28672x8192, 3INST k=2, batch 1, row-
    #      sharded over the ranks (all-gather of y~, replicated RHT-out); 4 distinct copies per shape in
    #      the graph (4 x 58.7 MB > L2).  Plus the all-gather latency of the exchange step alone.
    scaling_70b = None
    if not args.no_70b:
        scaling_70b = {"code": "3inst", "k": 2, "batch": 1, "ranks": world, "layers": {}}
        for si, (m, n) in enumerate([(8192, 28672), (28672, 8192)]):
            tiles = synth.random_tiles(m, n, 2, seed=1500 + si)
            smb, snb = synth.random_sign_bytes(m, 3501 + si), synth.random_sign_bytes(n, 3500 + si)
            copies = []
            for c in range(4):
                if world == 1:
                    lay = QTIPLinear(m, n, code="3inst", k=2, device=dev)
                    if c == 0:
                        lay.load_tiles(tiles, smb, snb)
                    else:
                        lay.packed.copy_(copies[0].packed)
                        lay.sign_m.copy_(copies[0].sign_m)
                        lay.sign_n.copy_(copies[0].sign_n)
                else:
                    lay = ShardedQTIPLinear(m, n, rank, world, code="3inst", k=2, device=dev)
                    if c == 0:
                        lay.load_tiles(tiles, smb, snb)
                    else:
                        lay.local.packed.copy_(copies[0].local.packed)
                        lay.local.sign_n.copy_(copies[0].local.sign_n)
                        lay.sign_m.copy_(copies[0].sign_m)
                copies.append(lay)
            del tiles
            xc = torch.from_numpy(synth.random_x(1, n, seed=2500 + si)).to(dev)
            yc = [torch.empty((1, m), dtype=torch.float32, device=dev) for _ in copies]
            loc = [(c if world == 1 else c.local) for c in copies]
            yl = [torch.empty((1, t.m), dtype=torch.float32, device=dev) for t in loc]

            def run_c4(gemv_only=False):
                for c, lay in enumerate(copies):
                    if gemv_only:
                        loc[c].forward(xc, out=yl[c], flags=qtip.QTIP_RHT_IN | qtip.QTIP_XT_READY)
                    elif world == 1:
                        lay.forward(xc, out=yc[c])
                    else:
                        yc[c].copy_(lay.forward(xc))

            times = {}
            for mode in (False, True):
                run_c4()
                gc = torch.cuda.CUDAGraph()
                with torch.cuda.stream(s):
                    run_c4(mode)
                    with torch.cuda.graph(gc, stream=s):
                        run_c4(mode)
                torch.cuda.current_stream().wait_stream(s)
                for _ in range(3):
                    gc.replay()
                barrier()
                c0_, c1_ = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                c0_.record()
                for _ in range(5):
                    gc.replay()
                c1_.record()
                torch.cuda.synchronize()
                times[mode] = max_over_ranks(1e3 * c0_.elapsed_time(c1_) / (5 * len(copies)))
                del gc
            scaling_70b["layers"][f"{m}x{n}"] = {
                "us_per_layer": round(times[False], 3), "GBps": round(m * n / 4 / (times[False] * 1e-6) / 1e9, 1),
                "gemv_only_us_max_over_ranks": round(times[True], 3),
                "rank_rows": (copies[0].rows[1] - copies[0].rows[0]) if world > 1 else m}
            del copies, loc
        if world > 1:
            lam = {}
            for nbytes_ag in (32768, 114688):
                per = nbytes_ag // 4 // world
                send_t = torch.zeros(per, dtype=torch.float32, device=dev)
                recv_t = torch.empty(per * world, dtype=torch.float32, device=dev)
                for _ in range(10):
                    dist.all_gather_into_tensor(recv_t, send_t)
                barrier()
                a0, a1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                a0.record()
                for _ in range(100):
                    dist.all_gather_into_tensor(recv_t, send_t)
                a1.record()
                torch.cuda.synchronize()
                lam[str(nbytes_ag)] = round(max_over_ranks(1e3 * a0.elapsed_time(a1) / 100), 3)
            scaling_70b["allgather_us"] = lam
        torch.cuda.empty_cache()

    cpu = None
    if world == 1 and rank == 0 and not args.no_cpu_baseline:
        cpu = cpu_baseline(code, k)

    path = "layers"
    if chain_res is not None:
        path = "chain"
        ms = chain_res["ms"]
        value = step_bytes / (ms * 1e-3) / 1e9
    sm_count = torch.cuda.get_device_properties(dev).multi_processor_count
    clk_sum = clk.summary()
    clk_mhz = clk_sum.get("sm_mhz") or 1965.0
    alu_bound = (code, k) == ("3inst", 2)
    alu_peak = 32 * sm_count * clk_mhz * 1e6 * k / 8 / 1e9            # GB/s of k-bit stream
    if rank == 0:
        line = {
            "metric": "fused trellis-decode GEMV: compressed-byte HBM GB/s vs peak; us/layer batch=1",
            "value": round(value, 2), "unit": "GB/s", "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": round(ms, 5), "higher_is_better": True, "scaling": "strong" if world > 1 else "weak",
            "vs_baseline": None, "dtype": "f16", "data": "synthetic",
            "config": {"workload": args.workload, "layers_per_step": len(layers), "blocks": nblocks,
                       "code": code, "k": k, "L": 16, "V": 2 if code == "hyb" else 1, "T": 256, "batch": B,
                       "stream_bytes_per_step": step_bytes, "tokens_per_s_equiv": round(B * 1e3 / ms, 2),
                       "per_layer": per_layer, "parallelism": f"rows{world}" if world > 1 else "single",
                       "path": path,
                       "dependency": ("chain: group g reads the output of one layer of group g-1 (o <- q, gate/up <- o, "
                                      "down <- gate, next q/k/v <- down); q,k,v and gate,up share an input"
                                      if chained else "fixed input per shape; groups sequential"),
                       "layers_path": layers_path,
                       "chain_stages": chain_res["stages"] if chain_res else None,
                       "grouping": args.grouping,
                       "step_serial_ms": round(ms_serial, 5),
                       "serial_GBps": round(step_bytes / (ms_serial * 1e-3) / 1e9, 2),
                       "l2": "inputs > L2: 1.62 GB of distinct packed weights per step (126 MB L2)"
                       if args.workload == "llama2-7b" else "distinct weights per layer",
                       "matvec_impl": qtip.get_matvec_impl(),
                       "arith": "decoded weights and RHT'd x in binary16, fp32 accumulation"},
            # against the MEASURED HBM copy bandwidth (MEASURED_PEAKS.json): the metric is compressed
            # bytes per second.  The integer-decode bounds of 3INST k=2 are context only.
            "roofline": {"bound": "hbm", "achieved": round(value if chain_res else gemv_gbs, 1), "peak": peak,
                         "unit": "GB/s", "frac": round((value if chain_res else gemv_gbs) / peak, 4),
                         "traffic": traffic(args.workload, code, k, qtip.get_matvec_impl()),
                         "kernel": ("chain_kernel: the step's single persistent launch (decode-GEMV of every layer + "
                                    "in-kernel RHTs), algorithmic stream bytes / its duration (one ~1 us counter memset "
                                    "per step included)" if chain_res else
                                    "fused decode-GEMV launches of the step (grouped where the step groups), back-to-back graph"),
                         "peak_kind": peak_kind,
                         "us_per_layer": round(1e3 * (ms if chain_res else gemv_ms / prof_steps) / len(layers), 3),
                         # context: the ALU-pipe bound of the 3INST k=2 decode (32 weights/clk/SM: per weight
                         # 1/2 funnel shift + 1/2 shift + 1 LOP3 at 64 lanes/clk/SM) and the measured
                         # decode + mma.sync loop ceiling (scripts/decode_microbench.cu, 19.2 weights/clk/SM)
                         "alu_bound": (None if not alu_bound else {
                             "GBps": round(alu_peak, 1), "frac": round(gemv_gbs / alu_peak, 4)}),
                         "decode_loop_ceiling": (None if (code, k) != ("3inst", 2) else {
                             "weights_per_clk_per_sm": 19.2, "GBps": round(19.2 * sm_count * clk_mhz * 1e6 * k / 8 / 1e9, 1),
                             "frac": round(gemv_gbs / (19.2 * sm_count * clk_mhz * 1e6 * k / 8 / 1e9), 4)})},
            "scaling_70b": scaling_70b,
            "cpu_baseline": cpu,
            "e2e": ({"value": round(step_bytes / (chain_res["e2e_ms"] * 1e-3) / 1e9, 2), "unit": "GB/s",
                     "h2d_bytes_per_step": chain_res["h2d"], "d2h_bytes_per_step": chain_res["d2h"],
                     "ms_per_step": round(chain_res["e2e_ms"], 5)} if chain_res else
                    {"value": round(step_bytes / (e2e_ms * 1e-3) / 1e9, 2), "unit": "GB/s", "h2d_bytes_per_step": h2d,
                     "d2h_bytes_per_step": d2h, "ms_per_step": round(e2e_ms, 5)}),
            "gpu_launches": (chain_res["launches"] if chain_res else launches_per_step) * args.steps,
            "clocks": clk_sum,
        }
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()


def relaunch_multi_rank(args):
    """`bench.py --gpus N` without torchrun: start N ranks on this node (torch.distributed.run, one
    process per GPU, rendezvous on 127.0.0.1) -- or fail clearly when fewer GPUs are visible."""
    import socket
    import torch
    ngpu = torch.cuda.device_count()
    if ngpu < args.gpus:
        raise SystemExit(f"bench.py: --gpus {args.gpus} but only {ngpu} CUDA device(s) visible")
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
           "--master-addr", "127.0.0.1", "--master-port", str(port), os.path.abspath(__file__)] + sys.argv[1:]
    os.execv(sys.executable, cmd)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--workload", default="llama2-7b", choices=sorted(WORKLOADS))
    ap.add_argument("--code", default=None, choices=["3inst", "1mad", "hyb"])
    ap.add_argument("--k", type=int, default=None)
    ap.add_argument("--batch", type=int, default=1)
    ap.add_argument("--blocks", type=int, default=None)
    ap.add_argument("--matvec-impl", type=int, default=0)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-70b", action="store_true", help="skip the C4 70B-layer block (scaling_70b)")
    ap.add_argument("--path", default="layers", choices=["chain", "layers"],
                    help="layers (default, measured fastest): per-layer RHT-in / GEMV / RHT-out launches; chain: "
                         "the whole step as one persistent chain-kernel launch (impl 8; 1 GPU, batch <= 16, chained "
                         "workloads; DESIGN.md 5.6)")
    ap.add_argument("--grouping", default="launch", choices=["streams", "launch", "serial"],
                    help="layers of a block that share an input: concurrent streams, one grouped launch, or serial")
    args = ap.parse_args()
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        relaunch_multi_rank(args)
    if args.impl == "reference":
        run_reference(args)
    else:
        run_ours(args)


if __name__ == "__main__":
    main()
