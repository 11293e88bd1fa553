"""Join FFB_GEMM_LOG shapes with an ncu launch list (same run order) -> per-shape GEMM time.
usage: python tools/gemm_table.py gemm_log.txt launches.csv"""
import csv
import re
import sys

lines = [l for l in open(sys.argv[2]) if l.startswith('"')]
seq = []
for r in csv.DictReader(lines):
    if r.get("Metric Name") != "gpu__time_duration.sum":
        continue
    v = float(r["Metric Value"].replace(",", ""))
    v *= {"ms": 1000.0, "ns": 1e-3}.get(r.get("Metric Unit"), 1.0)
    seq.append((r["Kernel Name"], v))
g = [l.strip()[7:] for l in open(sys.argv[1]) if l.startswith("[gemm]")]
out, gi, i = [], 0, 0
while i < len(seq):
    n, v = seq[i]
    if "gemm_f64_kernel" in n:
        if i + 1 < len(seq) and "splitk_reduce" in seq[i + 1][0]:
            v += seq[i + 1][1]
            i += 1
        out.append((g[gi] if gi < len(g) else "?", v))
        gi += 1
    i += 1
agg = {}
for sh, t in out:
    a = agg.setdefault(sh, [0, 0.0])
    a[0] += 1
    a[1] += t
tot = sum(t for _, t in out)
for sh, (c, t) in sorted(agg.items(), key=lambda kv: -kv[1][1])[:30]:
    M, N, K = map(int, re.findall(r"-?\d+", sh)[:3])
    print(f"{t:8.1f} us x{c:2d} {sh:55s} {2 * M * N * K * c / t / 1e6:6.1f} TF")
print(f"total GEMM {tot:.1f} us over {len(out)} launches; all kernels {sum(v for _, v in seq):.1f} us")
