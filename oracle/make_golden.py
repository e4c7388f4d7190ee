"""TEST-FIXTURE GENERATOR (run here, where /root/reference is mounted).

Produces tests/golden/ from the UNMODIFIED reference compiled by
oracle/Makefile (oracle/_ref/libcltkref.so):

* kernels/<name>.json -- kernelToJson of reindex(cutPayoff(compileContract(c)))
  (proj/src/kernel.cpp:620) for the five shipped contracts
  (proj/contracts/*.cl, read in place) and the two BASELINE contracts
  (contracts/worst-off.cl, contracts/brc.cl);
* models/<name>.json  -- model JSON (proj/README.md:85-94 schema);
* rng_kat.json        -- CounterRng bits/uniform/normal (proj/src/pricing.cpp:96-107);
* invnorm.json        -- invNormalCdf / normalCdf (proj/src/pricing.cpp:109-148);
* cases.json          -- pricing cases: priceAcrossTime prices/SE
  (proj/src/pricing.cpp:327), floats stored as float.hex (exact);
* paths/<case>.npz    -- first K paths: simulatePath ext, disc, per-day payoffs.

    python oracle/make_golden.py
"""
from __future__ import annotations

import json
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
sys.path.insert(0, HERE)
from oracle_py import Ref  # noqa: E402

REF_CONTRACTS = "/root/reference/proj/contracts"
GOLD = os.path.join(ROOT, "tests", "golden")

CONTRACTS = {
    "european-call": (os.path.join(REF_CONTRACTS, "european-call.cl"), {}),
    "barrier": (os.path.join(REF_CONTRACTS, "barrier.cl"), {}),
    "double-option": (os.path.join(REF_CONTRACTS, "double-option.cl"), {}),
    "fx-swap": (os.path.join(REF_CONTRACTS, "fx-swap.cl"), {}),
    "template-option": (os.path.join(REF_CONTRACTS, "template-option.cl"), {"t0": 10, "t1": 80}),
    "worst-off": (os.path.join(ROOT, "contracts", "worst-off.cl"), {}),
    "brc": (os.path.join(ROOT, "contracts", "brc.cl"), {}),
}

MODELS = {
    # proj/python/tests/test_smoke.py:45 (BS oracle 4.579032085233791)
    "call": {"rate": 0.05, "labels": {"AAPL": {"spot": 100.0, "vol": 0.2}}},
    "call_r0": {"rate": 0.0, "labels": {"AAPL": {"spot": 100.0, "vol": 0.2}}},
    "call_sigma0": {"rate": 0.05, "labels": {"AAPL": {"spot": 100.0, "vol": 0.0}}},
    # proj/tests/acceptance.cpp:254-257 (criterion 9)
    "barrier": {"rate": 0.03, "labels": {"AAPL": {"spot": 100.0, "vol": 0.25, "drift": 0.03}}},
    "double": {"rate": 0.01, "dayCount": 360.0,
               "labels": {"AAPL": {"spot": 100.0, "vol": 0.2},
                          "MSFT": {"spot": 250.0, "vol": 0.3, "drift": 0.02}},
               "corr": [[1.0, 0.8], [0.8, 1.0]]},
    "fx": {"rate": 0.02, "labels": {"EUR": {"spot": 1.0, "vol": 0.1}}},
    # SURVEY.md Appendix A
    "three": {"rate": 0.03,
              "labels": {"SX5E": {"spot": 3758.05, "vol": 0.19},
                         "N225": {"spot": 11840.0, "vol": 0.21},
                         "SPX": {"spot": 1200.0, "vol": 0.17}},
              "order": ["SX5E", "N225", "SPX"],
              "corr": [[1.0, 0.6, 0.5], [0.6, 1.0, 0.4], [0.5, 0.4, 1.0]]},
}

# name, kernel, model, seed, days, K (paths stored per path), price path counts
CASES = [
    ("call", "european-call", "call", 42, [0], 4096, [1, 1000, 100000, 1000000]),
    ("call_r0", "european-call", "call_r0", 42, [0], 256, [100000]),
    ("call_days", "european-call", "call", 5, [0, 45, 90, 91], 256, [20000]),
    ("call_sigma0", "european-call", "call_sigma0", 1, [0], 4, [1, 7]),
    ("barrier", "barrier", "barrier", 11, [0, 10], 1024, [50000]),
    ("double", "double-option", "double", 3, [0, 30, 45], 1024, [50000]),
    ("fxswap", "fx-swap", "fx", 1, [0, 30, 60, 90], 16, [1000]),
    ("template", "template-option", "call", 9, [0, 10, 50, 90, 91], 256, [20000]),
    ("worst_off", "worst-off", "three", 42, [0], 1024, [100000]),
    ("worst_off_days", "worst-off", "three", 7, [0, 100, 200, 300, 365, 366], 256, [20000]),
    ("brc", "brc", "three", 42, [0], 64, [2000]),
    ("brc_days", "brc", "three", 13, [0, 180, 366, 367], 16, [500]),
]

RNG_KAT = [(0, 0, 0), (0, 0, 1), (42, 0, 0), (42, 0, 1000), (7, 3, 0),
           (2**64 - 1, 123456789, 0), (1, 2**63, 5), (2**32 + 7, 2**40 + 3, 2**33 + 1)]


def hexf(x: float) -> str:
    return float(x).hex()


def main() -> None:
    sys.setrecursionlimit(1_000_000)
    ref = Ref()
    for sub in ("kernels", "models", "paths"):
        os.makedirs(os.path.join(GOLD, sub), exist_ok=True)

    kernels = {}
    for name, (path, tenv) in CONTRACTS.items():
        src = open(path).read()
        k = ref.compile_kernel(src, tenv, cut=True)
        kernels[name] = k
        with open(os.path.join(GOLD, "kernels", name + ".json"), "w") as f:
            json.dump(k, f, sort_keys=True)
        with open(os.path.join(GOLD, "kernels", name + ".kernel"), "w") as f:
            f.write(ref.kernel_source(k))
    for name, m in MODELS.items():
        with open(os.path.join(GOLD, "models", name + ".json"), "w") as f:
            json.dump(m, f, indent=1, sort_keys=True)

    rng = np.random.default_rng(2108_03076)
    kat = [{"seed": s, "path": p, "i": i} for (s, p, i) in RNG_KAT]
    for _ in range(200):
        kat.append({"seed": int(rng.integers(0, 2**63)), "path": int(rng.integers(0, 2**40)),
                    "i": int(rng.integers(0, 4096))})
    for e in kat:
        e["bits"] = "0x%016x" % ref.philox_bits(e["seed"], e["path"], e["i"])
        e["uniform"] = hexf(ref.uniform(e["seed"], e["path"], e["i"]))
        e["normal"] = hexf(ref.normal(e["seed"], e["path"], e["i"]))
    with open(os.path.join(GOLD, "rng_kat.json"), "w") as f:
        json.dump({"anchor": "Random123 philox2x64-10 KAT (ctr=0,key=0) = "
                             "{ca00a0459843d731, 66c24222c9a845b5}; c0^c1 = acc2e26751eb9284",
                   "kat": kat}, f, indent=0)

    ps = [1e-300, 1e-20, 1e-10, 1e-5, 0.001, 0.02, 0.02425, 0.024250000000000001, 0.1, 0.3,
          0.5, 0.7, 0.975, 0.97575, 0.99, 1 - 1e-10, float.fromhex("0x1.fffffffffffffp-1")]
    ps += [float(x) for x in rng.random(500)]
    ps += [float(x) for x in rng.random(200) * 0.02425]
    inv = [{"p": hexf(p), "x": hexf(ref.inv_normal_cdf(p))} for p in ps]
    cdf_x = [-38.0, -8.0, -6.0, -2.5, -0.3, 0.0, 0.7, 3.1, 4.0, 8.0]
    cdf = [{"x": hexf(x), "cdf": hexf(ref.normal_cdf(x))} for x in cdf_x]
    with open(os.path.join(GOLD, "invnorm.json"), "w") as f:
        json.dump({"inv": inv, "cdf": cdf, "domain_errors": [0.0, 1.0, -0.5, 1.5]}, f, indent=0)

    cases = []
    for (name, kname, mname, seed, days, K, counts) in CASES:
        k, m = kernels[kname], MODELS[mname]
        ext = ref.simulate_paths(k, m, seed, 0, K)
        disc = ref.disc(k, m)
        pay = ref.path_payoffs(k, m, seed, 0, K, days)
        np.savez_compressed(os.path.join(GOLD, "paths", name + ".npz"), ext=ext, disc=disc,
                            payoffs=pay, days=np.array(days, dtype=np.uint64))
        prices = []
        tenv = CONTRACTS[kname][1]
        for n in counts:
            res = ref.price(k, m, n, seed, days, tenv=tenv, threads=os.cpu_count())
            prices.append({"paths": n, "price": [hexf(r["price"]) for r in res],
                           "std_error": [hexf(r["std_error"]) for r in res],
                           "price_dec": [r["price"] for r in res]})
        cases.append({"name": name, "kernel": kname, "model": mname, "seed": seed, "days": days,
                      "tenv": tenv, "K": K, "prices": prices})
        print(name, [p["price_dec"] for p in prices])
    with open(os.path.join(GOLD, "cases.json"), "w") as f:
        json.dump({"cases": cases}, f, indent=1)


if __name__ == "__main__":
    main()
