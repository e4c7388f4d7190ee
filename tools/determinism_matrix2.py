"""Determinism matrix, part 2: template batches (both RNG modes), wide
models (9 / 17 / 32 assets, NVRTC), the remaining shipped contracts; repeated
launches, distinct results (1 expected) and NVRTC == interpreter where both run."""
import os
import sys

sys.path.insert(0, os.getcwd())
sys.path.insert(0, os.path.join(os.getcwd(), "tests"))
import paper_2108_03076_b200 as E  # noqa: E402
from conftest import load_model, load_kernel  # noqa: E402
from test_jit import _brc_batch_literals  # noqa: E402
from test_gpu_parity import _wide_model  # noqa: E402

reps = int(sys.argv[1]) if len(sys.argv) > 1 else 12


def run(label, f, modes=(False, True)):
    pats = {}
    for jit in modes:
        try:
            pats[jit] = {repr(f(jit)) for _ in range(reps)}
        except Exception as e:  # noqa: BLE001
            print(label, jit, "skip:", str(e)[:80], flush=True)
    ok = all(len(v) == 1 for v in pats.values())
    same = len(pats) < 2 or pats[False] == pats[True]
    print(label, {k: len(v) for k, v in pats.items()}, "OK" if ok and same else "FAIL", flush=True)


kj, lit = _brc_batch_literals(64)
for rng in ("philox", "sobol"):
    run(f"brc batch {rng}", lambda jit, rng=rng: [x[0]["price"] for x in
        E.price_template(kj, lit, load_model("three"), 20_064, 9, rng=rng, jit=jit)])
wo = load_kernel("worst-off")
wlit = E.kernel_literals(wo)
import numpy as np  # noqa: E402
wl = np.asarray([[v * (0.9 + 0.2 * i / 63) if v in (0.75, 1.0) else v for v in wlit] for i in range(64)])
for rng in ("philox", "sobol"):
    run(f"worst-off batch {rng}", lambda jit, rng=rng: [x[0]["price"] for x in
        E.price_template(wo, wl, load_model("three"), 200_064, 9, rng=rng, jit=jit)])
for na in (9, 17, 32):
    run(f"worst-off {na} assets", lambda jit, na=na: [x["price"] for x in
        E.price(E.Kernel(wo), _wide_model(na), 40_064, 9, [0, 150, 300], jit=jit)], modes=(True,))
for kname, mname, days in (("double-option", "double", [0, 30, 45]), ("template-option", "call", [0, 10, 50])):
    tenv = {"t0": 10, "t1": 80} if kname == "template-option" else None
    for rng in ("philox", "sobol"):
        run(f"{kname} {rng}", lambda jit, rng=rng: [x["price"] for x in
            E.price(E.Kernel(load_kernel(kname)), load_model(mname), 500_064, 9, days, tenv=tenv, rng=rng, jit=jit)])
