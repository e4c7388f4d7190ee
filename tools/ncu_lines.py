"""Per-source-line executed instructions and stall samples of an ncu capture
(the cuda+sass source page), for the NVRTC kernel whose sources are not on
this machine: python tools/ncu_lines.py <rep> <units> [top]"""
import csv
import io
import os
import subprocess
import sys

rep, units = os.path.abspath(sys.argv[1]), float(sys.argv[2])
top = int(sys.argv[3]) if len(sys.argv) > 3 else 60
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                     capture_output=True, text=True, cwd="/tmp").stdout
f = None
hdr = None
rows = []
for r in csv.reader(io.StringIO(out)):
    if not r:
        continue
    if r[0] == "File Path":
        f = r[1].split("/")[-1]
        continue
    if r[0] == "Line No":
        hdr = r
        continue
    if hdr and r[0].isdigit():
        d = dict(zip(hdr, r))
        rows.append((f, int(r[0]), int(d["# Samples"] or 0), int(d["Instructions Executed"] or 0)))
S = sum(x[2] for x in rows)
I = sum(x[3] for x in rows)
print(f"total samples {S}, warp instructions per unit {I / units * 32:.1f} (x32 lanes / unit)")
for f, ln, s, i in sorted(rows, key=lambda x: -x[2])[:top]:
    print(f"{f:22s} {ln:5d}  samples {100 * s / S:5.2f}%  inst/unit {32 * i / units:9.1f}")
