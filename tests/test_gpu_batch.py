"""Template batches of >= 32 instances (BASELINE config 4) reduce their outputs
instance-major (cltk_plan_header::inst_major): lane i sums instance i over the
warp's 32 paths in the order (jj + inst) mod 32.  The NVRTC kernel evaluates
the instance section per (path, instance) from the path's register columns,
the interpreter path-major with parked values -- the same values in the same
order, so the two payoff modes agree bitwise; against instances priced one
at a time (a different summation order) prices agree to the engine's stated
tolerance, and any sharding of the chunks gives the same bits.
"""
import pytest

import paper_2108_03076_b200 as E
from conftest import load_kernel, load_model

pytestmark = pytest.mark.gpu

PRICE_REL = 1e-13
SE_REL = 1e-9


def _table(kern, n):
    base = E.kernel_literals(kern)
    rows = []
    for i in range(n):
        b = 0.5 + 0.3 * i / max(1, n - 1)
        if kern["horizon"] > 300 and 2630.635 in base:  # BRC: barrier levels
            sub = {2630.635: 3758.05 * b, 8288.0: 11840.0 * b, 840.0: 1200.0 * b}
        else:  # worst-off: knock-in level
            sub = {0.75: b}
        rows.append([sub.get(v, v) for v in base])
    return rows


@pytest.mark.parametrize("kern,paths,n_inst", [("worst-off", 40_000, 100), ("brc", 3_000, 64),
                                               ("worst-off", 9_999, 33)])
def test_instance_major_batch_modes_bitwise_and_vs_single(kern, paths, n_inst):
    k = load_kernel(kern)
    m = load_model("three")
    lits = _table(k, n_inst)
    jit = E.price_template(k, lits, m, paths, 7, [0], jit=True)
    interp = E.price_template(k, lits, m, paths, 7, [0], jit=False)
    assert jit == interp
    for i in (0, 1, n_inst // 2, n_inst - 1):
        one = E.price_template(k, [lits[i]], m, paths, 7, [0])[0][0]
        got = jit[i][0]
        assert abs(got["price"] - one["price"]) <= PRICE_REL * abs(one["price"]), (i, got, one)
        assert abs(got["std_error"] - one["std_error"]) <= SE_REL * one["std_error"] + 1e-14


def test_instance_major_batch_is_shard_invariant():
    k = load_kernel("worst-off")
    m = load_model("three")
    lits = _table(k, 40)
    one = E.price_template(k, lits, m, 123_457, 3, [0])
    assert E.price_template(k, lits, m, 123_457, 3, [0], devices=[0, 0, 0]) == one


@pytest.mark.parametrize("kern,paths", [("worst-off", 20_000), ("brc", 2_000)])
def test_instance_major_batch_qmc_modes_bitwise(kern, paths):
    """The QMC mode's instance-major batches: the interpreter parks 16 rows
    (X, P and the bridge rows) instead of 12 -- still the same values in the
    same order as the NVRTC kernel."""
    k = load_kernel(kern)
    m = load_model("three")
    lits = _table(k, 40)
    jit = E.price_template(k, lits, m, paths, 5, [0], rng="sobol", jit=True)
    interp = E.price_template(k, lits, m, paths, 5, [0], rng="sobol", jit=False)
    assert jit == interp
    one = E.price_template(k, [lits[7]], m, paths, 5, [0], rng="sobol")[0][0]
    assert abs(jit[7][0]["price"] - one["price"]) <= PRICE_REL * abs(one["price"])


def test_stream_mode_multi_day_and_template_modes_bitwise():
    """Short paths (normal streams) with several valuation days and a small
    template table (< 32 instances: path-major reduction, parked in the P/Y
    rows while X still holds the stream's next normals)."""
    k = load_kernel("worst-off")
    m = load_model("three")
    lits = _table(k, 5)
    days = [0, 73, 200, 365]
    jit = E.price_template(k, lits, m, 50_001, 9, days, jit=True)
    interp = E.price_template(k, lits, m, 50_001, 9, days, jit=False)
    assert jit == interp
    for i in (0, 4):
        one = E.price_template(k, [lits[i]], m, 50_001, 9, days)[0]
        for a, b in zip(jit[i], one):
            assert a["price"] == b["price"] and a["std_error"] == b["std_error"]
