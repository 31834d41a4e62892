"""Summarise ncu reports (.ncu-rep) into the small text files committed under profiles/.

    python scripts/ncu_summary.py OUT.txt REPORT.ncu-rep [REPORT ...]
"""

from __future__ import annotations

import csv
import subprocess
import sys

KEYS = [
    ("gpu__time_duration.sum", "duration"),
    ("sm__cycles_elapsed.avg.per_second", "sm clock (cycles/s)"),
    ("dram__bytes_read.sum", "dram read"),
    ("dram__bytes_write.sum", "dram write"),
    ("gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "dram throughput % of peak"),
    ("lts__t_bytes.sum", "L2 bytes"),
    ("sm__inst_issued.avg.pct_of_peak_sustained_active", "issue slots busy %"),
    ("smsp__inst_executed.sum", "warp instructions executed"),
    ("sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active", "FMA pipe cycles active %"),
    ("sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_active", "ALU pipe cycles active %"),
    ("sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active", "XU (MUFU) pipe %"),
    ("sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active", "LSU pipe %"),
    ("sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active", "tensor pipe %"),
    ("launch__registers_per_thread", "registers/thread"),
    ("launch__grid_size", "grid"),
    ("launch__block_size", "block"),
    ("sm__warps_active.avg.pct_of_peak_sustained_active", "achieved occupancy %"),
    ("smsp__warps_active.avg.per_cycle_active", "active warps per scheduler"),
]


def summarise(path: str) -> list[str]:
    out = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(out.splitlines()))
    if len(rows) < 3:
        return [f"{path}: no data"]
    hdr, units = rows[0], rows[1]
    lines = []
    for vals in rows[2:]:
        d = dict(zip(hdr, vals))
        u = dict(zip(hdr, units))
        lines.append(f"== {d.get('Kernel Name', '?')}")
        lines.append(f"   report: {path}")
        for key, label in KEYS:
            if key in d:
                lines.append(f"   {label:34s} {d[key]} {u.get(key, '')}")
        stalls = []
        for h, v in d.items():
            if h.startswith("smsp__average_warps_issue_stalled_") and h.endswith("_per_issue_active.ratio"):
                try:
                    fv = float(v.replace(",", ""))
                except ValueError:
                    continue
                if fv >= 0.03:
                    stalls.append((fv, h[len("smsp__average_warps_issue_stalled_"):-len("_per_issue_active.ratio")]))
        lines.append("   stalls (warps per issue): " + ", ".join(f"{n}={v:.2f}" for v, n in sorted(stalls, reverse=True)))
    return lines


def main(argv):
    out = argv[1]
    lines = []
    for rep in argv[2:]:
        lines += summarise(rep)
    with open(out, "w") as fh:
        fh.write("\n".join(lines) + "\n")
    print("\n".join(lines))


if __name__ == "__main__":
    main(sys.argv)
