"""C5 sweep: paths 1e6 .. 1e10 in decades for C1-C3 on this
GPU (G = 1 here; bench.py under torchrun gives G > 1).  One bench line per
(workload, paths) appended to gpurun_out/sweep.jsonl.  Sizes whose step would
exceed ~25 s are skipped (BRC above 1e9)."""
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
RATE = {"call": 5.0e10, "worst_off": 3.6e9, "brc": 6.2e7}  # paths/s, to bound the sweep
out = os.path.join(ROOT, "gpurun_out", "sweep.jsonl")
os.makedirs(os.path.dirname(out), exist_ok=True)
for w in ("call", "worst_off", "brc"):
    for e in range(6, 11):
        n = 10 ** e
        if n / RATE[w] > 25:
            continue
        cmd = [sys.executable, os.path.join(ROOT, "bench.py"), "--workload", w, "--paths-per-gpu",
               str(n), "--steps", "2", "--warmup", "3", "--e2e-steps", "0", "--no-cpu-baseline"]
        r = subprocess.run(cmd, capture_output=True, text=True, timeout=900)
        line = r.stdout.strip().splitlines()[-1] if r.stdout.strip() else json.dumps(
            {"workload": w, "paths": n, "error": r.stderr[-500:]})
        d = json.loads(line)
        rec = {"workload": w, "paths": n, "value": d.get("value"), "ms_per_step": d.get("ms_per_step"),
               "kernel_ms": d.get("config", {}).get("kernel_ms"), "price": d.get("price"),
               "std_error": d.get("std_error"), "clocks": d.get("clocks")}
        with open(out, "a") as f:
            f.write(json.dumps(rec) + "\n")
        print(json.dumps(rec), flush=True)
