"""Worst-off, QMC, NVRTC, three valuation days: which chunks / outputs differ
between repeated launches (full last chunk and partial)."""
import os
import sys

sys.path.insert(0, os.getcwd())
sys.path.insert(0, os.path.join(os.getcwd(), "tests"))
import torch  # noqa: E402
import paper_2108_03076_b200 as E  # noqa: E402
from paper_2108_03076_b200.distributed import DistributedPricer  # noqa: E402
from conftest import load_model, load_kernel  # noqa: E402

m = load_model("three")
stream = torch.cuda.current_stream(0).cuda_stream
for paths in (1 << 20, (1 << 20) + 64):
    pr = DistributedPricer(E.Kernel(load_kernel("worst-off")), m, [0, 100, 300], device=0, rng="sobol", jit=True)
    cp, nc = pr.plan.chunking(paths)
    nout = pr.plan.n_outputs
    parts = pr.partials(paths)
    parts.zero_()
    pr.plan.launch(paths, 20, 0, nc, parts.data_ptr(), stream)
    torch.cuda.synchronize()
    ref = parts.clone()
    for it in range(20):
        parts.zero_()
        pr.plan.launch(paths, 20, 0, nc, parts.data_ptr(), stream)
        torch.cuda.synchronize()
        d = (parts.view(torch.int64) != ref.view(torch.int64)).view(nc, nout, 3)
        ch = torch.nonzero(d.any(dim=2).any(dim=1)).view(-1).tolist()
        if ch:
            outs = torch.nonzero(d.any(dim=2).any(dim=0)).view(-1).tolist()
            print(paths, "chunkPaths", cp, "nc", nc, "it", it, "chunks", len(ch), ch[:8], "outs", outs,
                  "ref", ref.view(nc, nout, 3)[ch[0]].tolist(), "got", parts.view(nc, nout, 3)[ch[0]].tolist(), flush=True)
    print(paths, "done", flush=True)
