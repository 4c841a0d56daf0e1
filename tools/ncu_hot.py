"""Hottest SASS instructions (warp-stall samples) of each kernel in an ncu
report (needs --import-source / -lineinfo builds for the source page).

    python tools/ncu_hot.py report.ncu-rep [top]
"""
import csv
import io
import subprocess
import sys


def main():
    path = sys.argv[1]
    top = int(sys.argv[2]) if len(sys.argv) > 2 else 30
    out = subprocess.run(["ncu", "-i", path, "--page", "source", "--csv"], capture_output=True,
                         text=True).stdout
    blocks, cur = [], None
    for row in csv.reader(io.StringIO(out)):
        if row and row[0] == "Kernel Name":
            cur = [row[1], None, []]
            blocks.append(cur)
        elif cur is not None and cur[1] is None:
            cur[1] = row
        elif cur is not None and row:
            cur[2].append(row)
    for name, hdr, rows in blocks:
        isrc = hdr.index("Source")
        isamp = hdr.index("Warp Stall Sampling (All Samples)")
        total = sum(int(r[isamp] or 0) for r in rows)
        stall_cols = [j for j, h in enumerate(hdr) if h.startswith("stall_") or "Stall" in h and
                      j != isamp and "Sampling" not in h]
        print(f"== {name}  ({len(rows)} SASS, {total} samples)")
        ranked = sorted(range(len(rows)), key=lambda k: -int(rows[k][isamp] or 0))[:top]
        for k in sorted(ranked):
            r = rows[k]
            print(f"{k:5d} {int(r[isamp] or 0) / max(total, 1) * 100:5.1f}%  {r[isrc].strip()[:70]}")


if __name__ == "__main__":
    main()
