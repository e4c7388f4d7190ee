"""Per-lane output values of the last chunk priced alone (CLTK_DEBUG_V build):
NVRTC vs interpreter."""
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
paths = int(sys.argv[1]) if len(sys.argv) > 1 else 40000
vals = {}
for jit in (True, False):
    pr = DistributedPricer(E.Kernel(_up_barrier_brc()), m, [0, 100, 300], device=0, rng="sobol", jit=jit)
    cp, nc = pr.plan.chunking(paths)
    buf = torch.zeros(nc * 9 + cp + 64, dtype=torch.float64, device="cuda:0")
    pr.plan.launch(paths, 20, nc - 1, nc, buf.data_ptr(), stream)
    torch.cuda.synchronize()
    vals[jit] = buf[nc * 9: nc * 9 + cp].tolist()
    print("jit" if jit else "interp", "chunk mean", buf.view(-1)[(nc - 1) * 9 + 1].item(), flush=True)
for i, (a, b) in enumerate(zip(vals[True], vals[False])):
    if a != b:
        print("lane", i, "jit", a, "interp", b, flush=True)
