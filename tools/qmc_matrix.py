"""QMC NVRTC determinism matrix: contract x valuation days, repeated full
launches with a partial last chunk; distinct last-chunk means seen."""
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
stream = torch.cuda.current_stream(0).cuda_stream
paths = int(sys.argv[1]) if len(sys.argv) > 1 else 341056
for name, kern in (("up", _up_barrier_brc()), ("down", load_kernel("brc")),
                   ("worst-off", load_kernel("worst-off"))):
    for days in ([0], [0, 100, 300]):
        for jit in (True, False):
            try:
                pr = DistributedPricer(E.Kernel(kern), m, days, device=0, rng="sobol", jit=jit)
            except Exception as e:  # noqa: BLE001
                print(name, days, jit, "skip", e)
                continue
            cp, nc = pr.plan.chunking(paths)
            seen = {}
            for it in range(40):
                parts = pr.partials(paths)
                parts.zero_()
                pr.plan.launch(paths, 20, 0, nc, parts.data_ptr(), stream)
                torch.cuda.synchronize()
                tot = parts.view(nc, -1, 3)[:, 0, :]
                v = (tot[:, 0] * tot[:, 1]).sum().item()
                seen[v] = seen.get(v, 0) + 1
            print(name, days, "jit" if jit else "interp", len(seen), "distinct", list(seen.values()), flush=True)
