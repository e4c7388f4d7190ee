"""The reference's reachable in-loop error, driven on the device.

``CounterRng::uniform`` (proj/src/pricing.cpp:100-103) returns exactly 1.0
when ``bits >> 11 == 2^53 - 1``, and ``invNormalCdf`` then throws
``EvalError("invNormalCdf domain error")`` (:111-113), which
``priceAcrossTime`` rethrows on the caller's thread (:345-364).  At 2^-53 per
draw it cannot be found by search, so plans built with ``fault=True`` carry a
test hook that forces the Philox word of one (path, draw) to all ones.  The
engine must raise the reference's error (code 5) for every payoff mode -- the
bytecode interpreter, the NVRTC kernel, and the NVRTC path batches of short
paths -- and must NOT raise for a draw the reference never makes (the
non-drawing day 0 of the BRC, a path beyond the run).
"""
import pytest
import torch

import paper_2108_03076_b200 as E
from conftest import load_kernel, load_model

pytestmark = pytest.mark.gpu


def _run(plan, paths, seed):
    _, nc = plan.chunking(paths)
    parts = torch.zeros(nc * plan.n_outputs * 3, dtype=torch.float64, device="cuda")
    st = torch.cuda.current_stream().cuda_stream
    plan.launch(paths, seed, 0, nc, parts.data_ptr(), st)
    return plan.finalize(paths, seed, parts.data_ptr(), st)


@pytest.mark.parametrize("kern,model,days,jit,path,draw", [
    ("worst-off", "three", [0, 100], False, 777, 7),     # interpreter
    ("worst-off", "three", [0, 100], True, 4095, 14),    # NVRTC, last draw of the path
    ("brc", "three", [0], True, 12345, 1097),           # NVRTC, 1098 draws
    ("brc", "three", [0], False, 3, 3),                 # interpreter, first drawing step
    ("european-call", "call", [0], True, 5000, 0),      # NVRTC path batches (6 paths/batch)
    ("european-call", "call", [0], False, 0, 0),        # interpreter, path 0
])
def test_domain_error_raises_like_reference(kern, model, days, jit, path, draw):
    k = E.Kernel(load_kernel(kern))
    m = load_model(model)
    plan = E.Plan(k, m, days, jit=jit, fault=True)
    paths = 20000 if kern == "brc" else 100_000
    clean = _run(plan, paths, 42)
    # the fault build prices the same bits as the product kernel when no fault is set
    assert clean == _run(E.Plan(k, m, days, jit=jit), paths, 42)
    plan.set_fault(path, draw)
    with pytest.raises(E.ContractError, match="invNormalCdf domain error") as ei:
        _run(plan, paths, 42)
    assert ei.value.code == 5
    # the error word is reset: the plan prices again once the fault is gone
    plan.set_fault(-1, 0)
    assert _run(plan, paths, 42) == clean


@pytest.mark.parametrize("jit", [False, True])
def test_draws_the_reference_never_makes_do_not_raise(jit):
    # BRC rows [366, 0, ..., 365]: sorted day 0 is a dt = 0 step, the reference
    # draws nothing there (pricing.cpp:226-231), so draw indices 0..2 are
    # never evaluated; a path past the end is never simulated
    k = E.Kernel(load_kernel("brc"))
    m = load_model("three")
    plan = E.Plan(k, m, [0], jit=jit, fault=True)
    clean = _run(plan, 5000, 7)
    for path, draw in ((10, 1), (4999, 2), (5000, 3), (123456, 3)):
        plan.set_fault(path, draw)
        assert _run(plan, 5000, 7) == clean, (path, draw)


def test_fault_hook_needs_a_fault_build_and_philox():
    k = E.Kernel(load_kernel("worst-off"))
    m = load_model("three")
    with pytest.raises(E.ContractUnsupportedError, match="fault"):
        E.Plan(k, m, [0]).set_fault(1, 1)
    with pytest.raises(E.ContractUnsupportedError, match="Philox"):
        E.Plan(k, m, [0], rng="sobol", fault=True)


def test_device_sobol_integers_bit_exact_vs_scipy():
    """The QMC generator's device integers (both the warp-cooperative
    skip-ahead the path kernel uses and the per-point form) equal
    scipy.stats.qmc.Sobol(scramble=False, bits=32) bit for bit, from point 0
    and after skip-ahead."""
    import numpy as np
    from scipy.stats import qmc
    for n0, n, d0, nd, aligned in ((0, 4096, 0, 64, True), (0, 2048, 1000, 100, True),
                                   ((1 << 20) + 96, 1024, 0, 32, True),
                                   ((1 << 20) + 96, 1024, 1090, 12, True),
                                   (12345, 777, 5, 20, False), (0, 100, 2040, 8, False)):
        got = E.debug_sobol(n0, n, d0, nd, aligned)
        s = qmc.Sobol(d0 + nd, scramble=False, bits=32)
        if n0:
            s.fast_forward(n0)
        want = np.round(s.random(n) * 2.0**32).astype(np.uint64)[:, d0:]
        assert np.array_equal(got.astype(np.uint64), want), (n0, d0)
