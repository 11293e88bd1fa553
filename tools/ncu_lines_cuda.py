"""Warp-stall samples per CUDA source line (all files) of one launch in an ncu
report:  python tools/ncu_lines_cuda.py report.ncu-rep [launch_skip] [N]"""
import csv
import io
import subprocess
import sys

rep = sys.argv[1]
skip = sys.argv[2] if len(sys.argv) > 2 else "0"
N = int(sys.argv[3]) if len(sys.argv) > 3 else 30
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass",
                      "--launch-skip", skip, "--launch-count", "1"], capture_output=True, text=True).stdout
fname = "?"
agg = {}
tot = 0.0
rows = list(csv.reader(io.StringIO(out)))
for r in rows:
    if not r:
        continue
    if r[0] == "File Path":
        fname = r[1].split("/")[-1]
        continue
    if r[0] in ("Function Name", "Line No") or len(r) < 5:
        continue
    if r[0] and r[2] == "-":          # a CUDA source line row
        try:
            v = float(r[4] or 0)
        except ValueError:
            continue
        key = (fname, int(r[0]), r[1].strip()[:70])
        agg[key] = agg.get(key, 0.0) + v
        tot += v
for (f, ln, src), v in sorted(agg.items(), key=lambda kv: -kv[1])[:N]:
    print(f"{100 * v / max(tot, 1):5.1f}% {f}:{ln:<5d} {src}")
