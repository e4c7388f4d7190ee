"""TEST-FIXTURE GENERATOR (run here, where /root/reference is mounted).

Reference results at the BASELINE configurations' path counts (BASELINE.md
section 3), from the UNMODIFIED reference compiled by oracle/Makefile
(oracle/_ref/libcltkref.so) -- priceAcrossTime (proj/src/pricing.cpp:327-371)
on all host threads, simulatePath (:311-316) and the per-path evalKernel loop
(:349-358):

* big.json -- prices / standard errors (float.hex, exact):
    BRC 3 x 367, seed 42, 100,000 and 1,000,000 paths;
    worst-off 3 x 5, seed 42, 1,000,000 and 16,000,000 paths;
    European call, seed 42, 1,000,000 paths (BASELINE config 1);
* paths/brc_10k.npz -- the first 10,000 BRC paths (seed 42): the per-path
  payoffs, and per path a 64-bit polynomial checksum of the bit patterns of
  ext[rows][cols] (88 MB of spots do not belong in git; the checksum pins
  every bit of them).

    python oracle/make_golden_big.py
"""
from __future__ import annotations

import json
import os
import sys
import time

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
sys.path.insert(0, HERE)
from oracle_py import Ref  # noqa: E402

GOLD = os.path.join(ROOT, "tests", "golden")
HASH_P = np.uint64(0x100000001B3)


def ext_checksums(ext: np.ndarray) -> np.ndarray:
    """Per path: sum_i bits(ext.flat[i]) * P^(i+1) mod 2^64 over the row-major
    ext[rows][cols] of that path (tests/test_gpu_big.py recomputes it from the
    device's spots)."""
    n = ext.shape[0]
    bits = np.ascontiguousarray(ext).reshape(n, -1).view(np.uint64)
    w = np.empty(bits.shape[1], dtype=np.uint64)
    acc = np.uint64(1)
    with np.errstate(over="ignore"):
        for i in range(bits.shape[1]):
            acc = acc * HASH_P
            w[i] = acc
        return (bits * w[None, :]).sum(axis=1, dtype=np.uint64)


def main() -> None:
    ref = Ref()
    load = lambda sub, n: json.load(open(os.path.join(GOLD, sub, n + ".json")))
    brc, wo, call = load("kernels", "brc"), load("kernels", "worst-off"), load("kernels",
                                                                              "european-call")
    three, mcall = load("models", "three"), load("models", "call")
    threads = os.cpu_count() or 1
    out = {"threads": threads, "prices": []}
    for name, k, m, seed, days, n in (("brc", brc, three, 42, [0], 100_000),
                                      ("brc", brc, three, 42, [0], 1_000_000),
                                      ("worst_off", wo, three, 42, [0], 1_000_000),
                                      ("worst_off", wo, three, 42, [0], 16_000_000),
                                      ("call", call, mcall, 42, [0], 1_000_000)):
        t0 = time.time()
        res = ref.price(k, m, n, seed, days, threads=threads)
        dt = time.time() - t0
        out["prices"].append({"name": name, "seed": seed, "days": days, "paths": n,
                              "price": [float(r["price"]).hex() for r in res],
                              "std_error": [float(r["std_error"]).hex() for r in res],
                              "price_dec": [r["price"] for r in res],
                              "seconds": round(dt, 2)})
        print(name, n, [r["price"] for r in res], f"{dt:.1f}s", flush=True)
    with open(os.path.join(GOLD, "big.json"), "w") as f:
        json.dump(out, f, indent=1)

    K, step = 10_000, 1_000
    sums, pays = [], []
    for p0 in range(0, K, step):
        ext = ref.simulate_paths(brc, three, 42, p0, step)
        sums.append(ext_checksums(ext))
        pays.append(ref.path_payoffs(brc, three, 42, p0, step, [0])[:, 0])
    np.savez_compressed(os.path.join(GOLD, "paths", "brc_10k.npz"),
                        ext_checksum=np.concatenate(sums), payoffs=np.concatenate(pays),
                        seed=np.uint64(42))
    print("brc_10k written")


if __name__ == "__main__":
    main()
