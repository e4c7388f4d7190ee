"""Uninitialised shared-memory hunt: NVRTC prices with the dynamic shared
memory pre-filled (CLTK_JIT_FLAGS=-DCLTK_SMEM_POISON=<pattern>) vs unfilled."""
import os
import sys

sys.path.insert(0, os.getcwd())
sys.path.insert(0, os.path.join(os.getcwd(), "tests"))
import paper_2108_03076_b200 as E  # noqa: E402
from conftest import load_model, load_kernel  # noqa: E402
from test_jit import _up_barrier_brc  # noqa: E402

m = load_model("three")
for name, kern in (("up", _up_barrier_brc()), ("down", load_kernel("brc"))):
    for rng in ("sobol", "philox"):
        for days in ([0, 100, 300], [0]):
            r = E.price(E.Kernel(kern), m, 40000, 20, days, rng=rng, jit=True)
            print(os.environ.get("CLTK_JIT_FLAGS", "-"), name, rng, days, [x["price"] for x in r], flush=True)
