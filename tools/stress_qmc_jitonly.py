"""NVRTC QMC up-and-in BRC (days 0/100/300) priced repeatedly: distinct prices seen."""
import os
import sys

sys.path.insert(0, os.getcwd())
sys.path.insert(0, os.path.join(os.getcwd(), "tests"))
import paper_2108_03076_b200 as E  # noqa: E402
from conftest import load_model  # noqa: E402
from test_jit import _up_barrier_brc  # noqa: E402

m = load_model("three")
k = E.Kernel(_up_barrier_brc())
seen = {}
for it in range(int(sys.argv[1])):
    p = E.price(k, m, 40000, 20, [0, 100, 300], rng="sobol", jit=True)[0]["price"]
    seen[p] = seen.get(p, 0) + 1
print(os.environ.get("CLTK_JIT_FLAGS", ""), seen, flush=True)
