"""Print the key metrics of ncu reports (details page), one column per report.

    python tools/ncu_summary.py a.ncu-rep [b.ncu-rep ...]
"""
import csv
import io
import subprocess
import sys

KEYS = ["Duration", "DRAM Throughput", "Memory Throughput", "Executed Instructions",
        "Issue Slots Busy", "Executed Ipc Active", "Registers Per Thread",
        "Dynamic Shared Memory Per Block", "Achieved Occupancy", "L1/TEX Hit Rate",
        "L2 Hit Rate", "Warp Cycles Per Issued Instruction", "Grid Size", "Block Size",
        "Cluster Size", "Max Active Clusters", "Local Memory Spilling Requests"]


def metrics(path):
    out = subprocess.run(["ncu", "-i", path, "--page", "details", "--csv"], capture_output=True,
                         text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    if not rows:
        return {}, ""
    hdr = rows[0]
    iname, iunit, ival = hdr.index("Metric Name"), hdr.index("Metric Unit"), hdr.index("Metric Value")
    res = {}
    kernel = rows[1][hdr.index("Kernel Name")] if len(rows) > 1 else ""
    for r in rows[1:]:
        if len(r) > ival and r[iname] in KEYS and r[iname] not in res:
            res[r[iname]] = f"{r[ival]} {r[iunit]}".strip()
    return res, kernel


def main():
    reps = [metrics(p) for p in sys.argv[1:]]
    for p, (_, k) in zip(sys.argv[1:], reps):
        print(f"{p}: {k[:100]}")
    for key in KEYS:
        vals = [m.get(key, "-") for m, _ in reps]
        if any(v != "-" for v in vals):
            print(f"{key:38s} " + " | ".join(f"{v:>18s}" for v in vals))


if __name__ == "__main__":
    main()
