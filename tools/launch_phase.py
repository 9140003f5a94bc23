"""Kernels of one path step in launch order from an ncu launch list
(gpu__time_duration.sum), between two kernel-name markers.

    python tools/launch_phase.py launches.csv [first_marker] [stop_marker]
"""
import csv
import re
import sys


def main(path, first="shifted_copy", stop="build_args"):
    with open(path) as f:
        lines = [ln for ln in f if ln.startswith('"')]
    r = csv.reader(lines)
    hdr = next(r)
    ki, vi, gi, si = (hdr.index(k) for k in ("Kernel Name", "Metric Value", "Grid Size", "Stream"))
    rows = []
    for row in r:
        name = re.sub(r"\(.*", "", row[ki]).replace("void unnamed>::", "").replace("unnamed>::", "")
        rows.append((name, row[gi], row[si], float(row[vi]) / 1000))
    idx = [i for i, x in enumerate(rows) if first in x[0]]
    j = idx[-1]
    tot = {}
    while j < len(rows) and stop not in rows[j][0]:
        print(f"{rows[j][3]:8.1f} us  str {rows[j][2]:>3s} grid {rows[j][1]:>14s}  {rows[j][0][:64]}")
        tot[rows[j][2]] = tot.get(rows[j][2], 0.0) + rows[j][3]
        j += 1
    print("per stream (us):", {k: round(v, 1) for k, v in tot.items()})


if __name__ == "__main__":
    main(*sys.argv[1:])
