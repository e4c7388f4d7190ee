"""Per-path payoffs of the last chunk (paths = 39936 + k, k active paths):
NVRTC vs interpreter, the chunk priced alone."""
import os
import sys

sys.path.insert(0, os.getcwd())
sys.path.insert(0, os.path.join(os.getcwd(), "tests"))
import torch  # noqa: E402
import paper_2108_03076_b200 as E  # noqa: E402
from paper_2108_03076_b200.distributed import DistributedPricer  # noqa: E402
from conftest import load_model  # noqa: E402
from test_jit import _up_barrier_brc  # noqa: E402

m = load_model("three")
stream = torch.cuda.current_stream(0).cuda_stream
res = {}
for jit in (True, False):
    pr = DistributedPricer(E.Kernel(_up_barrier_brc()), m, [0, 100, 300], device=0, rng="sobol", jit=jit)
    sums = []
    for k in range(1, 65):
        paths = 39936 + k
        cp, nc = pr.plan.chunking(paths)
        parts = pr.partials(paths)
        parts.zero_()
        pr.plan.launch(paths, 20, nc - 1, nc, parts.data_ptr(), stream)
        torch.cuda.synchronize()
        n, mean = parts.view(-1, 3, 3)[nc - 1][0][0].item(), parts.view(-1, 3, 3)[nc - 1][0][1].item()
        sums.append(n * mean)
    vals = [sums[0]] + [sums[i] - sums[i - 1] for i in range(1, 64)]
    res[jit] = vals
diff = [(i, round(a, 6), round(b, 6)) for i, (a, b) in enumerate(zip(res[True], res[False])) if abs(a - b) > 1e-6]
print("per-path differences (lane, jit, interp):", diff, flush=True)
