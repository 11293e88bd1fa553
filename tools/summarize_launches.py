"""Aggregate an ncu --csv launch list (gpu__time_duration.sum) per kernel family.

usage: python tools/summarize_launches.py gpurun_out/launches.csv [--skip-first N]
"""
import csv
import re
import sys
from collections import defaultdict


def family(name):
    n = re.sub(r"\(.*", "", name)
    n = re.sub(r"void ", "", n)
    m = re.match(r"(ffb::)?([a-zA-Z0-9_]+)(<.*>)?", n)
    base = m.group(2) if m else n
    if base == "gemm_f64_kernel":
        args = re.search(r"<(.*)>", name)
        return "gemm_f64<" + (args.group(1) if args else "") + ">"
    return base


def main(path, skip=0):
    rows = []
    with open(path) as f:
        lines = [l for l in f if l.startswith('"')]
    rd = csv.DictReader(lines)
    for r in rd:
        if r.get("Metric Name") != "gpu__time_duration.sum":
            continue
        v = float(r["Metric Value"].replace(",", ""))
        unit = r.get("Metric Unit", "ns")
        if unit == "usecond":
            v *= 1e3
        elif unit == "msecond":
            v *= 1e6
        rows.append((int(r["ID"]), r["Kernel Name"], v))
    rows = rows[skip:]
    tot = sum(v for _, _, v in rows)
    agg = defaultdict(lambda: [0, 0.0])
    for _, nm, v in rows:
        f = family(nm)
        agg[f][0] += 1
        agg[f][1] += v
    print(f"launches={len(rows)} total={tot/1e6:.3f} ms (serialised, cold-cache)")
    for f, (c, v) in sorted(agg.items(), key=lambda kv: -kv[1][1]):
        try:
            print(f"{v/1e6:9.3f} ms {100*v/tot:5.1f}%  x{c:4d}  {f[:110]}")
        except BrokenPipeError:
            sys.exit(0)


if __name__ == "__main__":
    skip = int(sys.argv[sys.argv.index("--skip-first") + 1]) if "--skip-first" in sys.argv else 0
    main(sys.argv[1], skip)
