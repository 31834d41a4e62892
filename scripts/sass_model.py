"""Per-pair FMA-pipe cost of each inner loop of the shipped kernels, read from
their SASS (cuobjdump), for bench.py's executed-instruction roofline.

    python scripts/sass_model.py [--write]   ->  profiles/sass_model.json

A loop is a backward branch whose body holds packed FP32 (FFMA2/FADD2/FMUL2).
On sm_100 a packed instruction keeps a sub-partition's FMA pipe busy for 2
cycles (32 lanes x 2 ops), a scalar FFMA/FADD/FMUL/IMAD for 1 (DESIGN.md §3,
scripts/microbench_gram3.cu).  FMA-pipe cycles per pair of a loop =
(2 * packed + scalar FMA-pipe instructions in the body) / (pairs one pass of
the body evaluates per lane: rows R x columns per step).  The loops are told
apart by their instruction mix:
  sum, tile-local Gram   7 FFMA2 : 3 FADD2 : 1 FMUL2 per row-step of 4 columns
  sum, direct formula    7 FFMA2 : 7 FADD2 : 1 FMUL2 (+2 FMNMX3: near chunks)
  count, Gram filter     3 FFMA2 + 1 FMNMX3 per row-step of 2 columns
"""

from __future__ import annotations

import json
import re
import subprocess
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent
LIB = ROOT / "paper_1901_11204_b200" / "libpaircount.so"
OUT = ROOT / "profiles" / "sass_model.json"

# kernel instances (template arguments <WARPS, R, W, DIRECT, FLAT, COMP, SORTED>)
KERNELS = {
    "sorted_sum": ("pairs_kernelILi4ELi8ELi256ELb1ELb1ELb0ELb1E", 8),
    "flat_sum": ("pairs_kernelILi4ELi8ELi256ELb1ELb1ELb0ELb0E", 8),
    "gram_count": ("pairs_kernelILi4ELi12ELi192ELb0ELb1ELb0ELb0E", 12),
}
FMA_SCALAR = ("FFMA", "FADD", "FMUL", "IMAD", "HFMA2")
PACKED = ("FFMA2", "FADD2", "FMUL2")


def function_sass(sass: str, mangled: str) -> list[tuple[int, str]]:
    out, on = [], False
    for line in sass.splitlines():
        if "Function : " in line:
            on = mangled in line
            continue
        if on:
            m = re.match(r"\s*/\*([0-9a-f]{4,})\*/\s+(.*?);", line)
            if m:
                out.append((int(m.group(1), 16), m.group(2)))
    return out


def opcode(text: str) -> str:
    return re.sub(r"^@!?U?P\w+\s+", "", text).split()[0].split(".")[0]


def loops(ins):
    idx = {a: i for i, (a, _) in enumerate(ins)}
    found = []
    for i, (a, t) in enumerate(ins):
        if opcode(t) != "BRA":
            continue
        m = re.search(r"(0x[0-9a-f]+)", t)
        if not m:
            continue
        tgt = int(m.group(1), 16)
        if tgt < a and tgt in idx:
            body = [opcode(x) for _, x in ins[idx[tgt]:i + 1]]
            ops = {}
            for o in body:
                ops[o] = ops.get(o, 0) + 1
            if sum(ops.get(p, 0) for p in PACKED) >= 8 and len(body) < 1000:
                found.append(ops)
    return found


def model(lib: Path = LIB) -> dict:
    sass = subprocess.run(["cuobjdump", "-sass", str(lib)], check=True, capture_output=True, text=True).stdout
    res = {"lib_bytes": lib.stat().st_size, "kernels": {}}
    for name, (mangled, rows) in KERNELS.items():
        ins = function_sass(sass, mangled)
        entry = {}
        for ops in loops(ins):
            ffma2, fadd2, fmul2 = (ops.get(p, 0) for p in PACKED)
            cycles = 2 * (ffma2 + fadd2 + fmul2) + sum(ops.get(s, 0) for s in FMA_SCALAR)
            if fmul2 and ffma2 == 7 * fmul2 and fadd2 == 3 * fmul2:
                kind, cols = "gram", 4 * fmul2 // rows      # one FMUL2 per row-step of 4 columns
            elif fmul2 and ffma2 == 7 * fmul2 and fadd2 == 7 * fmul2:
                kind, cols = ("near" if ops.get("FMNMX3", 0) or ops.get("FMNMX", 0) else "direct"), 4 * fmul2 // rows
            elif not fmul2 and not fadd2 and ffma2 and ops.get("FMNMX3", 0) * 3 == ffma2:
                kind, cols = "gram_filter", 2 * (ffma2 // 3) // rows
            else:
                continue
            pairs = rows * cols
            if kind in entry and entry[kind]["body_len"] <= sum(ops.values()):
                continue  # an enclosing loop (e.g. the Gram chunk's two halves): keep the innermost
            entry[kind] = {"fma_cycles_per_pair": cycles / pairs, "mufu_per_pair": ops.get("MUFU", 0) / pairs,
                           "issue_per_pair": sum(ops.values()) / pairs, "body": ops,
                           "body_len": sum(ops.values())}
        res["kernels"][name] = entry
    return res


if __name__ == "__main__":
    m = model()
    if "--write" in sys.argv:
        OUT.write_text(json.dumps(m, indent=1) + "\n")
    print(json.dumps({k: {p: round(v["fma_cycles_per_pair"], 4) for p, v in e.items()} for k, e in m["kernels"].items()},
                     indent=1))
