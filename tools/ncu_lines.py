"""Per-CUDA-source-line stall samples for a kernel in an ncu report (needs -lineinfo).
usage: python tools/ncu_lines.py rep.ncu-rep [N]"""
import csv, io, subprocess, sys
from collections import defaultdict
rep = sys.argv[1]
N = int(sys.argv[2]) if len(sys.argv) > 2 else 30
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout
lines = out.splitlines()
agg = defaultdict(float)
tot = 0.0
cur = ""
for blk_start, l in enumerate(lines):
    pass
i = 0
while i < len(lines):
    l = lines[i]
    if l.startswith('"File Path"'):
        cur = l.split(",", 1)[1].strip('"').split("/")[-1]
    if l.startswith('"Line No"'):
        j = i + 1
        while j < len(lines) and not lines[j].startswith('"File Path"') and not lines[j].startswith('"Function Name"') and not lines[j].startswith('"Kernel Name"'):
            j += 1
        rows = list(csv.reader(io.StringIO("\n".join(lines[i:j]))))
        hdr = rows[0]
        k = hdr.index("Warp Stall Sampling (All Samples)")
        last = ("", "")
        for r in rows[1:]:
            if r[0]:
                last = (r[0], r[1].strip()[:70])
            try:
                v = float(r[k] or 0)
            except (ValueError, IndexError):
                continue
            if v:
                agg[(cur, last[0], last[1])] += v
                tot += v
        i = j
        continue
    i += 1
for (f, ln, src), v in sorted(agg.items(), key=lambda kv: -kv[1])[:N]:
    print(f"{100*v/tot:5.1f}% {f}:{ln:5s} {src}")
