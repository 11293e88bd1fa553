"""ncu --set full report(s) -> profiles/<name>_traffic.json: DRAM bytes
(dram__bytes_read.sum + dram__bytes_write.sum) per launch, per kernel family,
plus duration and pipe utilisation — the `traffic` source of bench.py's
roofline.  When a family has several captured launches, the one named by
--pick family=substring (matched against the full kernel name) is used, else
the longest.

usage: python tools/ncu_traffic.py out.json rep.ncu-rep [...] [--pick gemm_f64_kernel=64, 144]
"""
import csv
import io
import json
import re
import subprocess
import sys

M = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
     "sm__inst_executed_pipe_tensor_subpipe_dmma.avg.pct_of_peak_sustained_active",
     "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
     "sm__throughput.avg.pct_of_peak_sustained_elapsed", "launch__grid_size"]

SCALE = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "nsecond": 1e-9, "usecond": 1e-6,
         "ns": 1e-9, "us": 1e-6, "ms": 1e-3, "s": 1.0,
         "msecond": 1e-3, "second": 1.0}


def family(name):
    n = name.replace("(anonymous namespace)::", "").replace("void ", "")
    n = re.sub(r"\(.*", "", n)
    n = re.sub(r"<.*", "", n)
    return n.split("::")[-1]


def rows(path):
    out = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv", "--metrics", ",".join(M)],
                         capture_output=True, text=True).stdout
    r = list(csv.reader(io.StringIO(out)))
    hdr, units = r[0], r[1]
    for line in r[2:]:
        d, u = dict(zip(hdr, line)), dict(zip(hdr, units))
        def val(mn):
            v = d.get(mn, "")
            try:
                x = float(v.replace(",", ""))
            except ValueError:
                return None
            return x * SCALE.get(u.get(mn, ""), 1.0)
        yield d["Kernel Name"], {
            "time_s": val(M[0]), "dram_read": val(M[1]), "dram_write": val(M[2]),
            "dmma_pct": val(M[3]), "dram_pct": val(M[4]), "sm_pct": val(M[5]), "grid": val(M[6])}


def main(argv):
    out_path, reps, picks = argv[0], [], {}
    i = 1
    while i < len(argv):
        if argv[i] == "--pick":
            k, v = argv[i + 1].split("=", 1)
            picks[k] = v
            i += 2
        else:
            reps.append(argv[i])
            i += 1
    res = {}
    for rp in reps:
        for name, m in rows(rp):
            fam = family(name)
            if fam in picks and picks[fam] not in name:
                continue
            prev = res.get(fam)
            if prev is None or (m["time_s"] or 0) > prev["time_s"]:
                res[fam] = {"dram_bytes": (m["dram_read"] or 0) + (m["dram_write"] or 0),
                            "time_s": m["time_s"], "dmma_pct": m["dmma_pct"], "dram_pct": m["dram_pct"],
                            "sm_pct": m["sm_pct"], "grid": m["grid"], "kernel": name[:160],
                            "source": rp.split("/")[-1]}
    with open(out_path, "w") as f:
        json.dump(res, f, indent=1)
    for k, v in res.items():
        print(k, v)


if __name__ == "__main__":
    main(sys.argv[1:])
