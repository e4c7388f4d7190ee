"""Summarise an ncu --set full capture of the path kernel: headline metrics,
stall reasons, and executed instructions / stall samples per SASS region
(regions split at BAR.SYNC and at the hottest branch targets).
    python tools/ncu_regions.py gpurun_out/<rep>.ncu-rep <units> [window]
units: the work units of the launch (draws, paths) to normalise by."""
import collections
import csv
import io
import re
import subprocess
import sys

rep, units = sys.argv[1], float(sys.argv[2])
win = int(sys.argv[3]) if len(sys.argv) > 3 else 48
raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True,
                     text=True).stdout
rows = list(csv.reader(io.StringIO(raw)))
d = dict(zip(rows[0], rows[2]))
for k in ("gpu__time_duration.sum", "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active",
          "smsp__issue_active.avg.pct_of_peak_sustained_active",
          "sm__warps_active.avg.pct_of_peak_sustained_active", "launch__registers_per_thread",
          "launch__occupancy_limit_registers", "launch__occupancy_limit_shared_mem",
          "sm__inst_executed.sum", "dram__bytes_read.sum", "dram__bytes_write.sum"):
    print(f"{k:65s} {d.get(k)}")
src = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(src)))
hdr = rows[1]
data = [r for r in rows[2:] if len(r) == len(hdr)]
ia, isrc, iex = hdr.index("Address"), hdr.index("Source"), hdr.index("Instructions Executed")
reasons = [h for h in hdr if h.startswith("stall_") and "Not Issued" not in h]
ri = {h: hdr.index(h) for h in reasons}
base = int(data[0][ia], 16)
recs = []
tot = collections.Counter()
for r in data:
    st = {h: int(r[ri[h]]) if r[ri[h]].isdigit() else 0 for h in reasons}
    tot.update(st)
    recs.append((int(r[ia], 16) - base, r[isrc].strip(), int(r[iex] or 0), st))
T = sum(tot.values())
print("stalls:", ", ".join(f"{h[6:]} {v / T * 100:.1f}%" for h, v in tot.most_common(8)))
E = sum(x[2] for x in recs)
print(f"warp instructions per unit: {E / units:.1f}")
ops = collections.Counter()
for off, s, e, st in recs:
    op = re.sub(r"^@!?U?P\w+\s+", "", s).split()[0].split(".")[0] if s else "?"
    ops[op] += e
print("mix per unit:", ", ".join(f"{o}:{c / units:.1f}" for o, c in ops.most_common(16)))
cuts = [0] + [off for off, s, e, st in recs if "BAR.SYNC" in s] + [recs[-1][0] + 16]
print("regions (split at barriers):")
for a, b in zip(cuts, cuts[1:]):
    seg = [x for x in recs if a <= x[0] < b]
    e = sum(x[2] for x in seg)
    smp = sum(sum(x[3].values()) for x in seg)
    if e / units < 0.5:
        continue
    o2 = collections.Counter()
    for off, s, ee, st in seg:
        op = re.sub(r"^@!?U?P\w+\s+", "", s).split()[0].split(".")[0] if s else "?"
        o2[op] += ee
    print(f"  {a:#07x}-{b:#07x}: {e / units:7.1f} inst/unit {smp / T * 100:5.1f}% samples | " +
          ", ".join(f"{o}:{c / units:.1f}" for o, c in o2.most_common(7)))
