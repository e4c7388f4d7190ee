"""Determinism matrix (Philox and QMC): contract x valuation days x payoff
mode, repeated full launches; distinct bit patterns of the chunk partials
(1 expected) and whether NVRTC equals the interpreter."""
import os
import sys

sys.path.insert(0, os.getcwd())
sys.path.insert(0, os.path.join(os.getcwd(), "tests"))
import torch  # noqa: E402
import paper_2108_03076_b200 as E  # noqa: E402
from paper_2108_03076_b200.distributed import DistributedPricer  # noqa: E402
from conftest import load_model, load_kernel  # noqa: E402
from test_jit import _brc_batch_literals  # noqa: E402

stream = torch.cuda.current_stream(0).cuda_stream
reps = int(sys.argv[1]) if len(sys.argv) > 1 else 20
cases = [("european-call", "call", 4_000_064), ("worst-off", "three", 1_000_064),
         ("brc", "three", 60_064), ("fx-swap", "fx", 1_000_064), ("barrier", "barrier", 1_000_064)]
for rng in ("philox", "sobol"):
    for kname, mname, paths in cases:
        for days in ([0], [0, 30, 60]):
            pats = {}
            for jit in (False, True):
                try:
                    pr = DistributedPricer(E.Kernel(load_kernel(kname)), load_model(mname), days,
                                           device=0, rng=rng, jit=jit)
                except Exception as e:  # noqa: BLE001
                    print(rng, kname, days, jit, "skip:", str(e)[:60], flush=True)
                    continue
                _, nc = pr.plan.chunking(paths)
                seen = set()
                for _ in range(reps):
                    parts = pr.partials(paths)
                    parts.zero_()
                    pr.plan.launch(paths, 9, 0, nc, parts.data_ptr(), stream)
                    torch.cuda.synchronize()
                    seen.add(hash(parts.view(torch.int64).cpu().numpy().tobytes()))
                pats[jit] = seen
            same = len(pats) == 2 and pats[False] == pats[True]
            print(rng, kname, days, {k: len(v) for k, v in pats.items()}, "jit==interp" if same else "DIFF", flush=True)
# template batches (NVRTC vs interpreter)
kj, lit = _brc_batch_literals(64)
for jit in (False, True):
    seen = set()
    for _ in range(max(4, reps // 4)):
        r = E.price_template(kj, lit, load_model("three"), 20_064, 9, jit=jit)
        seen.add(tuple(x[0]["price"] for x in r))
    print("brc batch", "jit" if jit else "interp", len(seen), flush=True)
