"""Small QMC / Philox runs for compute-sanitizer (racecheck / synccheck / initcheck):
the up-and-in BRC variant over three valuation days, both payoff modes."""
import os
import sys

sys.path.insert(0, os.getcwd())
sys.path.insert(0, os.path.join(os.getcwd(), "tests"))
import paper_2108_03076_b200 as E  # noqa: E402
from conftest import load_model  # noqa: E402
from test_jit import _up_barrier_brc  # noqa: E402

k = E.Kernel(_up_barrier_brc())
m = load_model("three")
for rng in ("sobol", "philox"):
    for jit in (False, True):
        r = E.price(k, m, int(sys.argv[1]) if len(sys.argv) > 1 else 2048, 7, [0, 100, 300],
                    rng=rng, jit=jit)
        print(rng, jit, [x["price"] for x in r], flush=True)
