"""Which payoff mode is nondeterministic: the same QMC up-and-in BRC price
(seed fixed) computed repeatedly by each mode."""
import os
import sys

sys.path.insert(0, os.getcwd())
sys.path.insert(0, os.path.join(os.getcwd(), "tests"))
import paper_2108_03076_b200 as E  # noqa: E402
from conftest import load_model  # noqa: E402
from test_jit import _up_barrier_brc  # noqa: E402

m = load_model("three")
k = E.Kernel(_up_barrier_brc())
n = int(sys.argv[1]) if len(sys.argv) > 1 else 30
days = [0] if len(sys.argv) > 2 and sys.argv[2] == "1" else [0, 100, 300]
for jit in (False, True):
    seen = {}
    for it in range(n):
        p = E.price(k, m, 40000, 20, days, rng="sobol", jit=jit)[0]["price"]
        seen[p] = seen.get(p, 0) + 1
    print("jit" if jit else "interp", seen, flush=True)
