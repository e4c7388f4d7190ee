"""Stress: template batches (NVRTC + interpreter) interleaved with the QMC
up-and-in BRC priced by both payoff modes; reports any NVRTC/interpreter
price mismatch (one was seen once in a GPU-suite run)."""
import os
import sys

sys.path.insert(0, os.getcwd())
sys.path.insert(0, os.path.join(os.getcwd(), "tests"))
import paper_2108_03076_b200 as E  # noqa: E402
from conftest import load_model  # noqa: E402
from test_jit import _brc_batch_literals, _up_barrier_brc  # noqa: E402

m = load_model("three")
kj, lit = _brc_batch_literals(40)
k = E.Kernel(_up_barrier_brc())
bad = 0
n = int(sys.argv[1]) if len(sys.argv) > 1 else 20
for it in range(n):
    E.price_template(kj, lit, m, 30000, 11 + it, jit=True)
    E.price_template(kj, lit, m, 30000, 11 + it, jit=False)
    for rng in ("sobol", "philox"):
        a = E.price(k, m, 40000, 7 + it, [0, 100, 300], rng=rng, jit=False)
        b = E.price(k, m, 40000, 7 + it, [0, 100, 300], rng=rng, jit=True)
        if [x["price"] for x in a] != [y["price"] for y in b]:
            bad += 1
            print("MISMATCH", it, rng, [x["price"] for x in a], [y["price"] for y in b], flush=True)
print(f"{bad} mismatches in {n} iterations", flush=True)
