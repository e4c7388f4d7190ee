"""Last-chunk probe: the NVRTC QMC plan's last (partial) chunk priced alone
(a fresh CTA) vs inside the full launch, and with many chunks per CTA."""
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
rng = sys.argv[1] if len(sys.argv) > 1 else "sobol"
for jit, paths in ((True, 40000), (False, 40000), (True, 888 * 128 * 3 + 64)):
    pr = DistributedPricer(E.Kernel(_up_barrier_brc()), m, [0, 100, 300], device=0, rng=rng, jit=jit)
    cp, nc = pr.plan.chunking(paths)
    parts = pr.partials(paths)
    last = nc - 1
    seen_full, seen_alone = {}, {}
    for it in range(60):
        parts.zero_()
        pr.plan.launch(paths, 20, 0, nc, parts.data_ptr(), stream)
        torch.cuda.synchronize()
        v = parts.view(-1, 3, 3)[last][0][1].item()
        seen_full[v] = seen_full.get(v, 0) + 1
        parts.zero_()
        pr.plan.launch(paths, 20, last, nc, parts.data_ptr(), stream)
        torch.cuda.synchronize()
        v = parts.view(-1, 3, 3)[last][0][1].item()
        seen_alone[v] = seen_alone.get(v, 0) + 1
    print(rng, "jit" if jit else "interp", paths, "chunks", nc, "chunkPaths", cp, "full:", seen_full, "alone:", seen_alone, flush=True)
