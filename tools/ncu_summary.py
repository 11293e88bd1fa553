"""One line per captured launch of an ncu --set full report: duration, DRAM
traffic, DMMA (FP64 tensor) pipe utilisation, DRAM throughput, SM throughput.

usage: python tools/ncu_summary.py report.ncu-rep [more.ncu-rep ...]"""
import csv
import io
import subprocess
import sys

METRICS = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
           "sm__inst_executed_pipe_tensor_subpipe_dmma.avg.pct_of_peak_sustained_active",
           "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
           "sm__throughput.avg.pct_of_peak_sustained_elapsed", "launch__grid_size"]
SHORT = ["time", "dram_rd", "dram_wr", "dmma%", "dram%", "sm%", "grid"]


def main(paths):
    for p in paths:
        out = subprocess.run(["ncu", "-i", p, "--page", "raw", "--csv", "--metrics", ",".join(METRICS)],
                             capture_output=True, text=True).stdout
        rows = list(csv.reader(io.StringIO(out)))
        hdr, units = rows[0], rows[1]
        for r in rows[2:]:
            d, u = dict(zip(hdr, r)), dict(zip(hdr, units))
            name = d["Kernel Name"].split("(")[0].replace("void ", "")[:58]
            vals = " ".join(f"{s}={d.get(m, '?')}{u.get(m, '')}" for s, m in zip(SHORT, METRICS))
            print(f"{name:58s} {vals}")


if __name__ == "__main__":
    main(sys.argv[1:])
