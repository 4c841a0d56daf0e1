"""Selected raw metrics of an ncu report, one column per kernel launch.

    python tools/ncu_raw.py report.ncu-rep [metric-substring ...]
"""
import csv
import io
import subprocess
import sys

DEFAULT = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
           "dram__throughput.avg.pct_of_peak_sustained_elapsed",
           "sm__inst_executed.sum", "sm__issue_active.avg.pct_of_peak_sustained_active",
           "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active",
           "sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active",
           "smsp__average_warp_latency_issue_stalled",
           "smsp__average_warps_issue_stalled_", "launch__registers_per_thread",
           "sm__warps_active.avg.pct_of_peak_sustained_active",
           "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum",
           "local_"]


def main():
    path = sys.argv[1]
    keys = sys.argv[2:] or DEFAULT
    out = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True,
                         text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr, units, data = rows[0], rows[1], rows[2:]
    ik = hdr.index("Kernel Name")
    print("kernel:", " | ".join(r[ik][:50] for r in data))
    for j, h in enumerate(hdr):
        if any(k in h for k in keys):
            vals = [r[j] for r in data]
            if h.startswith("smsp__average_warps_issue_stalled_"):
                try:
                    if max(float(v.replace(",", "")) for v in vals) < 0.05:
                        continue
                except ValueError:
                    pass
            print(f"{h} [{units[j]}]: " + " | ".join(vals))


if __name__ == "__main__":
    main()
