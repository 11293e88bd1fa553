"""Top stall lines of an ncu report's source page: python tools/ncu_source_hot.py rep.ncu-rep [N]"""
import csv
import io
import subprocess
import sys

rep = sys.argv[1]
N = int(sys.argv[2]) if len(sys.argv) > 2 else 25
view = sys.argv[3] if len(sys.argv) > 3 else "source"
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", view],
                     capture_output=True, text=True).stdout
lines = out.splitlines()
start = [i for i, l in enumerate(lines) if l.startswith('"Address"') or l.startswith('"Line"') or l.startswith('"#"')]
rows = list(csv.reader(io.StringIO("\n".join(lines[start[0]:]))))
hdr = rows[0]
ix = {h: i for i, h in enumerate(hdr)}
k = ix["Warp Stall Sampling (All Samples)"]
src = ix["Source"]
stall_cols = [h for h in hdr if h.startswith("stall_") and "Not Issued" not in h]
data = []
for r in rows[1:]:
    try:
        v = float(r[k] or 0)
    except ValueError:
        continue
    top = sorted(((float(r[ix[h]] or 0), h) for h in stall_cols), reverse=True)[:2]
    data.append((v, r[src][:90], top))
tot = sum(d[0] for d in data) or 1
for v, s, top in sorted(data, key=lambda d: -d[0])[:N]:
    print(f"{100*v/tot:5.1f}%  {s:90s} {[(h[6:], int(x)) for x, h in top]}")
