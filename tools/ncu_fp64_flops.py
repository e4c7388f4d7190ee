"""Executed FP64 flops per unit of a captured path kernel, from the ncu source
page (predicated-on thread instructions of every DADD / DMUL / DFMA; DFMA = 2
flops):  python tools/ncu_fp64_flops.py <rep> <units>"""
import csv
import io
import re
import subprocess
import sys

rep, units = sys.argv[1], float(sys.argv[2])
src = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(src)))
hdr = rows[1]
ip = hdr.index("Predicated-On Thread Instructions Executed")
isrc = hdr.index("Source")
c = {"DADD": 0, "DMUL": 0, "DFMA": 0}
for r in rows[2:]:
    if len(r) != len(hdr):
        continue
    op = re.sub(r"^@!?U?P\w+\s+", "", r[isrc].strip()).split(" ")[0].split(".")[0]
    if op in c:
        c[op] += int(r[ip] or 0)
flops = c["DADD"] + c["DMUL"] + 2 * c["DFMA"]
print({k: v / units for k, v in c.items()}, "flops/unit", flops / units)
