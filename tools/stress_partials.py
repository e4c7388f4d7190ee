"""Nondeterminism hunt: the NVRTC QMC up-and-in BRC plan launched repeatedly;
per-chunk partials compared bitwise with the first launch (which chunks and
outputs differ, if any)."""
import os
import sys

sys.path.insert(0, os.getcwd())
sys.path.insert(0, os.path.join(os.getcwd(), "tests"))
import torch  # noqa: E402
import paper_2108_03076_b200 as E  # noqa: E402
from paper_2108_03076_b200.distributed import DistributedPricer  # noqa: E402
from conftest import load_model, load_kernel  # noqa: E402
from test_jit import _up_barrier_brc  # noqa: E402

m = load_model("three")
n = int(sys.argv[1]) if len(sys.argv) > 1 else 100
rng = sys.argv[2] if len(sys.argv) > 2 else "sobol"
k = E.Kernel(_up_barrier_brc())
pr = DistributedPricer(k, m, [0, 100, 300], device=0, rng=rng, jit=True)
other = DistributedPricer(E.Kernel(load_kernel("brc")), m, [0], device=0, rng="philox", jit=False)
paths, seed = int(os.environ.get("NPATHS", "40000")), 20
ref = pr.launch(paths, seed).clone()
torch.cuda.synchronize()
bad = 0
for it in range(n):
    other.price(20000, it)  # a different kernel in between
    p = pr.launch(paths, seed)
    torch.cuda.synchronize()
    if not torch.equal(p.view(torch.int64), ref.view(torch.int64)):
        bad += 1
        d = (p.view(torch.int64) != ref.view(torch.int64)).view(-1, 3, 3)  # [chunk][out][n,mean,m2]
        chunks = torch.nonzero(d.any(dim=2).any(dim=1)).view(-1).tolist()
        outs = torch.nonzero(d.any(dim=2).any(dim=0)).view(-1).tolist()
        print(f"it {it}: {len(chunks)} chunks differ {chunks[:10]}, outputs {outs}", flush=True)
        for c in chunks[:3]:
            print("  ref", ref.view(-1, 3, 3)[c].tolist(), "\n  got", p.view(-1, 3, 3)[c].tolist(), flush=True)
print(f"{bad} differing launches of {n} ({rng})", flush=True)
