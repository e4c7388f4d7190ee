#!/usr/bin/env python
"""Benchmark: Monte Carlo paths/s of the barrier reverse convertible
(3 underlyings x 367 dates, contracts/brc.cl; BASELINE.json metric) on
1..8 B200s, with the FP64 roofline fraction and the reference CPU pricer
timed beside it.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl b200|reference]

A step = one full pricing pass (simulate + payoff + reduce) over
paths_per_gpu * N paths of the BRC kernel (weak scaling), inputs (the compiled
program) resident on the device.  N > 1 runs one process per GPU under
torch.distributed (NCCL); the only data-path collective is the single
all-gather of the chunk partials.  `--gpus N` without torchrun re-launches
itself under `torch.distributed.run --nproc-per-node N`.  Rank 0 prints ONE
JSON line.
"""
from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)
sys.setrecursionlimit(100000)

METRIC = "MC paths/sec at 1/2/4/8 B200 (barrier reverse convertible), % FP roofline"
GOLD = os.path.join(ROOT, "tests", "golden")

# FP64 flops per path of the fused kernel, frozen from the ncu SASS op counters
# (dadd + dmul + 2*dfma) of the first correct kernel (profiles/).
F_PATH = {"brc": 286221.4, "worst_off": 3069.1, "call": 202.1, "brc_batch": 243.9,
          "worst_off_batch": 9.6}
# brc: ncu r1 (profiles/r1_path_kernel_brc_2M_raw.csv), 2e6 paths:
#   dadd 6.2471e10 + dmul 7.0817e10 + 2 * dfma 2.19577e11 thread-instructions
# worst_off / call: first measurement (profiles/r1_fp64ops_*_2M.csv), 2e6 paths
# C4 batches: FP64 flops per INSTANCE-path (1024 instances share each path),
# first measurement (profiles/r2a_fp64ops_*_batch_200k.csv, 2e5 paths x 1024):
#   brc_batch: dadd 8.8802e9 + dmul 1.15312e10 + 2 * dfma 1.47653e10 -> 243.9
#   worst_off_batch: dadd 8.2388e8 + dmul 5.9430e8 + 2 * dfma 2.7376e8 -> 9.6
# QMC mode (Sobol + AS241 + bridge) has its own F_path, frozen from the first
# measurement (profiles/r1_fp64ops_qmc_brc_2M.csv, 2e6 paths):
#   dadd 1.61651e10 + dmul 1.73608e10 + 2 * dfma 8.59067e10 thread-instructions
F_PATH_QMC = {"brc": 102669.7}

# DRAM bytes per launch of the path kernel from the committed ncu --set full
# capture (dram__bytes_read.sum + dram__bytes_write.sum; the kernel reads only
# its ~90 KB program and the partials stay in L2), and the FP64 pipe activity
# ncu measured there -- the kernel's own pipe utilisation beside the frozen-F
# roofline fraction.
# executed_f_path: FP64 flops per path the current kernel executes (ncu source
# page, predicated-on DADD + DMUL + 2 DFMA thread instructions,
# tools/ncu_fp64_flops.py) -- the second roofline figure beside the frozen one.
NCU_EVIDENCE = {
    "brc": {"traffic": 208384.0, "fp64_pipe_active": 0.486, "executed_f_path": 173142.4,
            "capture": "profiles/r2h_path_kernel_brc_10M_{raw.csv,summary.txt} (10M-path launch)"},
    "worst_off": {"traffic": 63232.0, "fp64_pipe_active": 0.470, "executed_f_path": 2732.4,
                  "capture": "profiles/r2h_path_kernel_worst_off_4M_{raw.csv,summary.txt}"},
    "call": {"traffic": 49664.0, "fp64_pipe_active": 0.429, "executed_f_path": 180.9,
             "capture": "profiles/r2h_path_kernel_call_40M_{raw.csv,summary.txt}"},
}

BATCH_N = 1024


def batch_literals(kern_json: str, workload: str = "brc_batch"):
    """C4: 1024 instances of one template, literal pool only.  BRC: knock-in
    barrier at 50%..80% of spot and strike at 90%..110% of spot; worst-off:
    knock-in level 0.50..0.80 and autocall trigger 0.90..1.10."""
    import paper_2108_03076_b200 as E
    base = E.kernel_literals(kern_json)
    rows = []
    for i in range(BATCH_N):
        b = 0.5 + 0.3 * i / (BATCH_N - 1)
        r = 0.9 + 0.2 * ((i * 389) % BATCH_N) / (BATCH_N - 1)
        sub = {}
        if workload == "brc_batch":
            spots = {3758.05: 2630.635, 11840.0: 8288.0, 1200.0: 840.0}  # spot -> 70% barrier
            for sp, bar in spots.items():
                sub[bar] = sp * b
                sub[sp] = sp * r
        else:
            sub[0.75] = b
            sub[1.0] = r
        rows.append([sub.get(v, v) for v in base])
    import numpy as np
    return np.asarray(rows, dtype=np.float64)  # the host table a caller hands in


WORKLOADS = {
    "brc_batch": ("brc", "three", f"C4: {BATCH_N} instances of the BRC template (barrier "
                  "50-80%, strike 90-110% of spot) on one path set, literals as kernel data"),
    "worst_off_batch": ("worst-off", "three", f"C4: {BATCH_N} instances of the worst-off template "
                        "(knock-in 0.50-0.80, autocall trigger 0.90-1.10) on one path set"),
    "brc": ("brc", "three", "BRC 3 underlyings x 367 dates (contracts/brc.cl, SURVEY.md App. A)"),
    "worst_off": ("worst-off", "three", "worst-off autocallable 3 x 5 dates (contracts/worst-off.cl)"),
    "call": ("european-call", "call", "European call 1 x 1 date (proj/contracts/european-call.cl)"),
}


def load(workload: str):
    kname, mname, desc = WORKLOADS[workload]
    kern = open(os.path.join(GOLD, "kernels", kname + ".json")).read()
    model = open(os.path.join(GOLD, "models", mname + ".json")).read()
    return kern, model, desc


class ClockSampler:
    """nvidia-smi clocks + throttle reasons sampled DURING the timed region."""

    Q = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.hw_slowdown,"
         "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
         "clocks_event_reasons.sw_power_cap")

    def __init__(self, gpu: int):
        self.gpu = gpu
        self.proc = None
        self.lines: list[str] = []
        self.t = None

    def start(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.gpu), f"--query-gpu={self.Q}",
                 "--format=csv,noheader,nounits", "-lms", "200"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except FileNotFoundError:
            self.proc = None

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def stop(self) -> dict:
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except Exception:
            self.proc.kill()
        if self.t:
            self.t.join(timeout=2)
        sm, mx, pw, reasons = [], [], [], set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in self.lines:
            f = [x.strip() for x in ln.split(",")]
            if len(f) < 7:
                continue
            try:
                sm.append(float(f[0]))
                mx.append(float(f[1]))
                pw.append(float(f[2]))
            except ValueError:
                continue
            for n, v in zip(names, f[3:7]):
                if v.lower().startswith("active"):
                    reasons.add(n)
        sm.sort()
        return {"sm_mhz": sm[len(sm) // 2] if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "power_w_max": max(pw) if pw else None, "samples": len(sm),
                "reasons": sorted(reasons)}


def cpu_reference(kern_json: str, model_json: str, paths: int, seed: int, threads: int):
    """The reference's own CPU pricer (oracle/_ref: the unmodified reference
    compiled from its sources) when present, else the C restatement."""
    sys.path.insert(0, os.path.join(ROOT, "oracle"))
    import oracle_py as O
    kern, model = json.loads(kern_json), json.loads(model_json)
    if O.ref_available():
        ref, kind = O.Ref(), "reference"
        t0 = time.perf_counter()
        r = ref.price(kern, model, paths, seed, [0], threads=threads)
    else:
        ref, kind = O.Oracle(), "port"
        t0 = time.perf_counter()
        r = ref.price(kern, model, paths, seed, [0], threads=threads)
    dt = time.perf_counter() - t0
    return kind, dt, r[0]


def run_reference_arm(args, rank: int):
    if rank != 0:
        return
    kern, model, desc = load(args.workload)
    threads = os.cpu_count() or 1
    sample = args.ref_paths
    for _ in range(args.warmup):
        cpu_reference(kern, model, sample, 42, threads)
    times = []
    res = None
    for _ in range(args.steps):
        kind, dt, res = cpu_reference(kern, model, sample, 42, threads)
        times.append(dt)
    t = sum(times) / len(times)
    v = sample / t
    line = {"impl": "reference", "metric": METRIC, "value": v, "unit": "paths/s",
            "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": t * 1e3, "higher_is_better": True, "scaling": "weak",
            "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": {"workload": desc, "paths_per_step": sample, "seed": 42,
                       "engine": "reference priceMC, std::thread over host cores"},
            "cpu_baseline": {"value": v, "unit": "paths/s", "cores": threads, "kind": kind,
                             "sample": f"{sample} paths of the same workload per step"},
            "e2e": {"value": v, "unit": "paths/s", "h2d_bytes_per_step": 0,
                    "d2h_bytes_per_step": 0},
            "price": res["price"], "std_error": res["std_error"]}
    print(json.dumps(line), flush=True)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="b200", choices=["b200", "reference"])
    ap.add_argument("--workload", default="brc", choices=sorted(WORKLOADS))
    ap.add_argument("--paths-per-gpu", type=int, default=125_000_000)
    ap.add_argument("--ref-paths", type=int, default=100_000)
    ap.add_argument("--e2e-steps", type=int, default=3)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--rng", default="philox", choices=["philox", "sobol"],
                    help="philox: the reference's generator (bit-exact parity); sobol: QMC mode")
    ap.add_argument("--jit", default="1", choices=["0", "1", "auto"],
                    help="payoff evaluation: 0 bytecode interpreter, 1 NVRTC-generated kernel "
                         "(bit-identical results)")
    args = ap.parse_args()
    args.jit = {"0": False, "1": True, "auto": "auto"}[args.jit]

    # the e2e calls build their plan every time (parse, compile, upload): no
    # in-process plan cache between timed calls
    os.environ["CLTK_PLAN_CACHE"] = "0"
    if args.gpus < 1:
        ap.error("--gpus must be >= 1")
    if args.impl == "b200" and args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        # one process per GPU: re-launch under torchrun (the driver's own launch
        # already sets WORLD_SIZE)
        import socket
        sk = socket.socket()
        sk.bind(("127.0.0.1", 0))
        port = sk.getsockname()[1]
        sk.close()
        argv = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1",
                f"--nproc-per-node={args.gpus}", "--master-addr", "127.0.0.1",
                "--master-port", str(port), os.path.abspath(__file__)] + sys.argv[1:]
        os.execv(sys.executable, argv)
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if args.impl == "reference":
        run_reference_arm(args, rank)
        return
    if world != args.gpus:
        raise SystemExit(f"bench: --gpus {args.gpus} but WORLD_SIZE {world}: launch one "
                         "process per GPU (torchrun --nproc-per-node N) or drop WORLD_SIZE")

    import torch
    import torch.distributed as dist
    import paper_2108_03076_b200 as E
    from paper_2108_03076_b200.distributed import DistributedPricer, gather_partials_

    visible = torch.cuda.device_count()
    if local >= visible:
        raise SystemExit(f"bench: rank {rank} needs GPU {local} but only {visible} visible")
    torch.cuda.set_device(local)
    if world > 1:
        dist.init_process_group("nccl", device_id=torch.device(f"cuda:{local}"))
    kern_json, model_json, desc = load(args.workload)
    kern = E.Kernel(kern_json)
    paths = args.paths_per_gpu * world
    seed = 42
    literals = (batch_literals(kern_json, args.workload) if args.workload.endswith("_batch")
                else None)
    n_inst = len(literals) if literals is not None else 1
    pricer = DistributedPricer(kern, model_json, [0], device=local, literals=literals, rng=args.rng,
                               jit=args.jit)
    info = pricer.plan.info
    dev = torch.device(f"cuda:{local}")
    flush = torch.empty(256 * 1024 * 1024 // 4, dtype=torch.float32, device=dev)  # > 126 MB L2

    def barrier():
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize(dev)

    # FP64 peak on this GPU (DFMA microbenchmark, burst)
    peak_tflops, _ = E.fp64_peak(local, 8192)

    for _ in range(args.warmup):
        pricer.finalize(paths, seed, pricer.launch(paths, seed))
    # multi-GPU: every rank must price the same bits as one GPU would
    check = pricer.finalize(paths, seed, pricer.launch(paths, seed))
    barrier()
    clocks = ClockSampler(local)
    clocks.start()
    time.sleep(1.5)  # nvidia-smi start-up (NVML init) outside the timed steps
    step_ms = []
    kernel_ms = []
    res = None
    stream = torch.cuda.current_stream(dev)
    for _ in range(args.steps):
        flush.fill_(1.0)  # L2 flush between timed steps (outside the events)
        barrier()
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        e2 = torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        parts = pricer.launch_local(paths, seed, stream.cuda_stream)  # this rank's chunk slice
        e1.record(stream)
        gather_partials_(parts)  # the one data-path collective (NCCL all-gather)
        res = pricer.finalize(paths, seed, parts)  # combine + read-back (synchronises)
        e2.record(stream)
        e2.synchronize()
        step_ms.append(e0.elapsed_time(e2))
        kernel_ms.append(e0.elapsed_time(e1))
    barrier()
    clk = clocks.stop()
    t_step = sum(step_ms) / len(step_ms)
    t_kern = sum(kernel_ms) / len(kernel_ms)
    if world > 1:
        tt = torch.tensor([t_step, t_kern], dtype=torch.float64, device=dev)
        dist.all_reduce(tt, op=dist.ReduceOp.MAX)
        t_step, t_kern = float(tt[0]), float(tt[1])
    value = paths * n_inst / (t_step * 1e-3)  # instance-paths/s (= paths/s for one contract)

    # end to end through the public API, host JSON in -> host results out; one
    # untimed call first (process-level caches: CUDA context, NVRTC module)
    e2e_times = []
    clocks_e2e = ClockSampler(local)
    clocks_e2e.start()
    time.sleep(1.5)  # nvidia-smi start-up (NVML init) outside the timed calls
    for it in range(args.e2e_steps + (1 if args.e2e_steps else 0)):
        barrier()
        t0 = time.perf_counter()
        if world > 1:
            from paper_2108_03076_b200 import distributed as D
            D.price(E.Kernel(kern_json), model_json, paths, seed, literals=literals, rng=args.rng,
                    jit=args.jit)
        elif literals is not None:
            E.price_template(kern_json, literals, model_json, paths, seed, rng=args.rng,
                             jit=args.jit)
        else:
            E.price(kern_json, model_json, paths, seed, rng=args.rng, jit=args.jit)
        torch.cuda.synchronize(dev)
        if it:
            e2e_times.append(time.perf_counter() - t0)
    clk_e2e = clocks_e2e.stop()
    # median of the timed calls (a host-side hiccup in one call does not move it)
    t_e2e = sorted(e2e_times)[len(e2e_times) // 2] if e2e_times else 0.0
    if world > 1:
        tt = torch.tensor([t_e2e], dtype=torch.float64, device=dev)
        dist.all_reduce(tt, op=dist.ReduceOp.MAX)
        t_e2e = float(tt[0])
    if [r["price"] for r in res] != [r["price"] for r in check]:
        raise SystemExit("bench: timed step priced different bits than the check step")
    # our kernels per timed step: the path kernel + the fixed-order combine
    # (two launches when the chunk count is split, engine_launch.hpp kCombineSplit)
    n_chunks = pricer.plan.chunking(paths)[1]
    n_launches = 1 + (2 if (n_chunks + 4095) // 4096 > 1 else 1)
    L = pricer.plan.dump()
    step_bytes = 32 + 24 * ((max(1, L["n_assets"]) + 1) // 2 * 2)  # device step records
    h2d = (len(L["ops"]) * 8 + len(L["steps"]) * step_bytes
           + (L["n_shared_const"] + L["n_inst_const"]) * 8
           + len(L["outputs"]) * 8 + 16 + len(kern_json) * 0)
    d2h = info["n_outputs"] * 24 + 8

    # roofline: FP64 pipe (the kernel reads only constants; no HBM term)
    fpath = F_PATH.get(args.workload) if args.rng == "philox" else F_PATH_QMC.get(args.workload)
    per_gpu_paths = paths / world
    if fpath:
        achieved = per_gpu_paths * n_inst * fpath / (t_kern * 1e-3) / 1e12
        ev = NCU_EVIDENCE.get(args.workload) if args.rng == "philox" and n_inst == 1 else None
        roof = {"bound": "fp64", "achieved": achieved, "peak": peak_tflops, "unit": "TFLOP/s",
                "frac": achieved / peak_tflops, "traffic": ev["traffic"] if ev else None,
                "peak_source": "measured DFMA microbenchmark (cltk_fp64_peak), this GPU, burst",
                "f_path": fpath}
        if ev:
            ach_x = per_gpu_paths * ev["executed_f_path"] / (t_kern * 1e-3) / 1e12
            roof.update({"traffic_unit": "bytes per launch", "ncu_capture": ev["capture"],
                         "fp64_pipe_active_ncu": ev["fp64_pipe_active"],
                         "achieved_basis": "frozen algorithmic F_path (first correct kernel) x "
                                           "paths/s; executed: the flops this kernel runs",
                         "executed_f_path": ev["executed_f_path"],
                         "achieved_executed": ach_x, "frac_executed": ach_x / peak_tflops})
    else:
        roof = {"bound": "fp64", "achieved": None, "peak": peak_tflops, "unit": "TFLOP/s",
                "frac": None, "traffic": None,
                "peak_source": "measured DFMA microbenchmark (cltk_fp64_peak), this GPU, burst",
                "f_path": None, "note": "F_path not yet frozen from ncu"}

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline and literals is None:
        threads = os.cpu_count() or 1
        kind, dt, r = cpu_reference(kern_json, model_json, args.ref_paths, seed, threads)
        one = max(1000, args.ref_paths // max(1, threads))
        _, dt1, _ = cpu_reference(kern_json, model_json, one, seed, 1)
        cpu = {"value": args.ref_paths / dt, "unit": "paths/s", "cores": threads, "kind": kind,
               "sample": f"{args.ref_paths} paths of the same workload, seed {seed}, "
                         f"{dt:.2f} s on {threads} threads",
               "value_1_thread": one / dt1,
               "seconds_for_1e9_paths": 1e9 * dt / args.ref_paths,
               "note": "1e9-path time extrapolated linearly from the sample",
               "price": r["price"], "std_error": r["std_error"]}

    if rank == 0:
        line = {"metric": METRIC, "value": value, "unit": "paths/s", "n_gpus": world,
                "steps": args.steps, "warmup": args.warmup, "ms_per_step": t_step,
                "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
                "data": "synthetic",
                "config": {"workload": desc, "instances": n_inst, "paths_per_gpu": args.paths_per_gpu,
                           "paths_per_step": paths, "seed": seed,
                           "rng": "philox2x64-10 (reference generator, bit-exact)" if args.rng == "philox"
                           else "sobol (Joe-Kuo) + AS241 + Brownian bridge (QMC)",
                           "payoff": "NVRTC-generated sm_100a kernel" if info["jit"]
                           else "bytecode interpreter (ahead-of-time kernel)",
                           "parallelism": f"paths sharded over {world} GPU(s) (one process "
                                          "each), 1 NCCL all-gather of the chunk partials",
                           "l2": "flushed between timed steps (256 MiB write); inputs are a "
                                 f"{h2d} B compiled program",
                           "kernel_ms": t_kern},
                "roofline": roof, "cpu_baseline": cpu,
                "e2e": {"value": paths * n_inst / t_e2e if t_e2e > 0 else None, "unit": "paths/s",
                        "h2d_bytes_per_step": h2d, "samples_ms": [round(t * 1e3, 3) for t in e2e_times],
                        "statistic": "median of the timed calls",
                        "plan_cache": "off (every call parses, compiles and uploads its plan)",
                        "d2h_bytes_per_step": d2h, "clocks": clk_e2e,
                        "path": "paper_2108_03076_b200.price -> cltk_gpu_price[_ex] (C-ABI), host "
                                "kernel/model JSON in, host results out"},
                "gpu_launches": n_launches, "clocks": clk,
                "price": res[0]["price"], "std_error": res[0]["std_error"],
                "plan": {k: info[k] for k in ("n_shared_ops", "n_thread", "dag_nodes", "jit")}}
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
