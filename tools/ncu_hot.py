"""Hot SASS lines (warp-stall samples) of one kernel in an ncu report.
usage: python tools/ncu_hot.py rep.ncu-rep kernel_regex [N]"""
import csv, io, subprocess, sys
rep, kre = sys.argv[1], sys.argv[2]
N = int(sys.argv[3]) if len(sys.argv) > 3 else 25
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass",
                      "-k", "regex:" + kre, "--launch-count", "1"], capture_output=True, text=True).stdout
lines = out.splitlines()
st = [i for i, l in enumerate(lines) if l.startswith('"Address"')][0]
end = [i for i, l in enumerate(lines) if l.startswith('"Kernel Name"') and i > st]
rows = list(csv.reader(io.StringIO("\n".join(lines[st:(end[0] if end else len(lines))]))))
hdr = rows[0]; ix = {h: i for i, h in enumerate(hdr)}
K = ix["Warp Stall Sampling (All Samples)"]
stalls = [h for h in hdr if h.startswith("stall_") and "Not" not in h]
tot = sum(float(r[K] or 0) for r in rows[1:]) or 1
tot_st = {h: sum(float(r[ix[h]] or 0) for r in rows[1:]) for h in stalls}
print("samples", tot, "| stall mix:", ", ".join(f"{h[6:]}={100*v/tot:.0f}%" for h, v in sorted(tot_st.items(), key=lambda kv: -kv[1])[:6]))
for r in sorted(rows[1:], key=lambda r: -float(r[K] or 0))[:N]:
    v = float(r[K] or 0)
    top = sorted(((float(r[ix[h]] or 0), h) for h in stalls), reverse=True)[:2]
    print(f"{100*v/tot:5.1f}% {r[ix['Address']][-5:]} {r[ix['Source']][:58]:58s} {[(h[6:], int(x)) for x, h in top]}")
