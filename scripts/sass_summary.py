#!/usr/bin/env python
"""Per-weight SASS instruction mix of each hot decode-GEMV kernel in libqtip.so (no GPU needed).

For a kernel instance, the decode loop is the innermost loop (backward branch) holding the most
weight-consuming instructions -- STTM (tcgen05.st of the decoded A operand, impl 7) or HMMA
(register-fed mma.sync, impls 3-6).  Its instructions are counted by opcode and class and divided
by the weights one thread handles per iteration:
    STTM.x8 = 8 TMEM columns x 2 binary16 weights = 16 weights per thread;
    HMMA.16816 = 256 A elements per warp = 8 weights per lane (HYB) or 4 (K-doubled 3INST / 1MAD).

usage: python scripts/sass_summary.py [out_dir]
"""
import collections
import os
import re
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
LIB = os.path.join(ROOT, "paper_2406_11235_b200", "libqtip.so")

# (label, mangled-name regex, weights per STTM/HMMA, code)
KERNELS = [
    ("impl7_3inst_k2", r"umma_gemv_kernelILi2ELi2ELi16ELb1E", 16, "3inst"),
    ("impl7_hyb_k4", r"umma_gemv_kernelILi4ELi3ELi16ELb0E", 16, "hyb"),
    ("impl7_hyb_k3", r"umma_gemv_kernelILi3ELi3ELi16ELb0E", 16, "hyb"),
    ("impl6_3inst_k2", r"layer_kernelILi2ELi2ELb1E", 4, "3inst"),
    ("impl6_hyb_k4", r"layer_kernelILi4ELi3ELb0E", 8, "hyb"),
    ("impl4_3inst_k2", r"gemv_row_kernelILi2ELi2ELb1E", 4, "3inst"),
    ("impl4_hyb_k4", r"gemv_row_kernelILi4ELi3ELb0E", 8, "hyb"),
    ("impl3_3inst_k2", r"gemv_mma_kernelILi2ELi2ELi1E", 4, "3inst"),
]
CLASSES = {
    "alu": {"LOP3", "SHF", "PRMT", "IADD3", "LEA", "SEL", "ISETP", "PLOP3", "VIADD", "IMNMX", "VIMNMX", "FLO", "POPC",
            "BMSK", "SGXT", "LOP"},
    "fma": {"IMAD", "IDP", "HADD2", "HFMA2", "HMUL2", "FFMA", "FADD", "FMUL"},
    "lsu": {"LDS", "STS", "LDG", "STG", "LDL", "STL", "LDSM", "ATOMS", "LD", "ST"},
    "tensor": {"HMMA", "UTCHMMA", "STTM", "LDTM"},
    "uniform": set(),
    "sync/branch": {"BRA", "BAR", "SYNCS", "BSSY", "BSYNC", "WARPSYNC", "NOP", "EXIT", "YIELD", "ELECT", "VOTE", "VOTEU"},
}


def cls(op):
    base = op.split(".")[0]
    if base.startswith("U") and base not in ("UTCHMMA",):
        return "uniform"
    for c, s in CLASSES.items():
        if base in s:
            return c
    return "other"


def sass(fn):
    out = subprocess.run(["cuobjdump", "-sass", "-fun", fn, LIB], capture_output=True, text=True).stdout
    ins = []
    for line in out.splitlines():
        m = re.match(r"\s+/\*([0-9a-f]+)\*/\s+(@!?U?P\w+\s+)?([A-Z][A-Z0-9_.]*)(.*);", line)
        if m:
            ins.append((int(m.group(1), 16), m.group(3), m.group(4)))
    return ins


def functions():
    out = subprocess.run(["cuobjdump", "-sass", LIB], capture_output=True, text=True).stdout
    return sorted(set(re.findall(r"Function : (\S+)", out)))


def loop_body(ins, marker):
    loops = []
    for addr, op, rest in ins:
        if op.startswith("BRA"):
            m = re.search(r"0x([0-9a-f]+)", rest)
            if m and int(m.group(1), 16) < addr:
                loops.append((int(m.group(1), 16), addr))
    best = None
    for lo, hi in loops:
        body = [(a, o) for a, o, _ in ins if lo <= a <= hi]
        nm = sum(1 for _, o in body if o.split(".")[0] == marker)
        if nm == 0:
            continue
        key = (-(hi - lo), nm)                     # the innermost loop holding the marker
        if best is None or key > best[0]:
            best = (key, body)
    return best[1] if best else []


def main():
    out_dir = sys.argv[1] if len(sys.argv) > 1 else os.path.join(ROOT, "profiles", "r2")
    os.makedirs(out_dir, exist_ok=True)
    fns = functions()
    summary = []
    for label, pat, wper, code in KERNELS:
        cands = [f for f in fns if re.search(pat, f)]
        if not cands:
            summary.append(f"{label}: not found")
            continue
        fn = cands[0]
        ins = sass(fn)
        marker = "STTM" if label.startswith("impl7") else "HMMA"
        body = loop_body(ins, marker)
        nmark = sum(1 for _, o in body if o.split(".")[0] == marker)
        weights = nmark * wper
        ops = collections.Counter(o.split(".")[0] for _, o in body)
        by = collections.Counter(cls(o) for _, o in body)
        lines = [f"{label}  ({fn})", f"decode loop: {len(body)} instructions, {nmark} {marker} -> {weights} weights per "
                 f"thread per iteration -> {len(body) / max(weights, 1):.2f} instructions per weight"]
        lines.append("by class (per weight): " + ", ".join(f"{c} {n / max(weights, 1):.2f}" for c, n in by.most_common()))
        lines.append("by opcode (count): " + ", ".join(f"{o} {n}" for o, n in ops.most_common()))
        with open(os.path.join(out_dir, f"sass_{label}.txt"), "w") as f:
            f.write("\n".join(lines) + "\n")
        summary.append(lines[1].replace("decode loop", label) + " | " + lines[2])
    with open(os.path.join(out_dir, "sass_summary.txt"), "w") as f:
        f.write("\n".join(summary) + "\n")
    print("\n".join(summary))


if __name__ == "__main__":
    main()
