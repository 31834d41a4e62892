"""Summarise an ncu launch list (--metrics gpu__time_duration.sum --csv) into profiles/*_summary.txt:
the kernels of the first 2^20 step (prep_bbox_kernel .. finalize_kernel) with their shares, then the
per-kernel totals of the whole command.

    python scripts/launch_summary.py LAUNCHES.csv OUT.txt "header line"
"""
import csv
import io
import sys
from collections import defaultdict


def short(name: str) -> str:
    return name.split("(")[0] if not name.startswith("void ") else name.split("(")[0]


def main():
    src, out, header = sys.argv[1], sys.argv[2], sys.argv[3]
    text = open(src).read()
    text = text[text.index('"ID"'):]
    rows = [r for r in csv.DictReader(io.StringIO(text)) if r["Metric Name"] == "gpu__time_duration.sum"]
    scale = {"ns": 1e-6, "us": 1e-3, "usecond": 1e-3, "ms": 1.0, "msecond": 1.0, "nsecond": 1e-6}
    launches = [(short(r["Kernel Name"]), float(r["Metric Value"].replace(",", "")) * scale[r["Metric Unit"]]) for r in rows]
    i0 = next(i for i, (k, _) in enumerate(launches) if "prep_bbox_kernel" in k)
    i1 = next(i for i in range(i0, len(launches)) if "finalize_kernel" in launches[i][0])
    step = launches[i0:i1 + 1]
    tot = sum(t for _, t in step)
    lines = [header, "per-launch times are cold-cache and serialised; the shares of one 2^20 step are what must agree with the live timing",
             "", "one 2^20 step (first call):"]
    lines += [f"  {k[:60]:<60} {t:9.3f} ms {100 * t / tot:6.1f} %" for k, t in step]
    lines.append(f"  total {tot:.3f} ms")
    agg = defaultdict(float)
    for k, t in launches:
        agg[k] += t
    all_t = sum(agg.values())
    lines += ["", "all launches of the command (incl. the e2e calls and the cfg4 2^22 leg):"]
    lines += [f"  {k[:60]:<60} {t:10.2f} ms {100 * t / all_t:6.1f} %" for k, t in sorted(agg.items(), key=lambda x: -x[1])[:12]]
    open(out, "w").write("\n".join(lines) + "\n")
    print("\n".join(lines[:30]))


if __name__ == "__main__":
    main()
