"""Models wider than 16 assets (CLTK_MAX_ASSETS=32 build): NVRTC prices vs the
oracle (pinned to the reference) within the summation-order tolerance."""
import os
import sys

sys.path.insert(0, os.getcwd())
sys.path.insert(0, os.path.join(os.getcwd(), "tests"))
sys.path.insert(0, os.path.join(os.getcwd(), "oracle"))
import paper_2108_03076_b200 as E  # noqa: E402
from conftest import load_kernel  # noqa: E402
from oracle_py import Oracle  # noqa: E402
from test_gpu_parity import _wide_model  # noqa: E402

for n_assets, kern, days, n in ((17, "worst-off", [0, 150], 4000), (24, "worst-off", [0], 4000),
                                (32, "worst-off", [0, 300], 2000), (20, "brc", [0], 200)):
    k, m = load_kernel(kern), _wide_model(n_assets)
    want = Oracle().price(k, m, n, 5, days, threads=os.cpu_count() or 1)
    got = E.price(E.Kernel(k), m, n, 5, days)
    for x, w in zip(got, want):
        rel = abs(x["price"] - w["price"]) / abs(w["price"])
        print(n_assets, kern, days, x["price"], w["price"], "rel %.2e" % rel, flush=True)
