"""Parity at the BASELINE configurations' path counts, against fixtures the
UNMODIFIED reference produced (oracle/make_golden_big.py, committed with its
outputs tests/golden/big.json and tests/golden/paths/brc_10k.npz), and --
where the compiled reference travelled with the repo (oracle/_ref) --
against the reference itself on the box.

Tolerances (tests/test_gpu_parity.py): per-path spots and payoffs bit-exact;
prices |dP| <= 1e-13 |P| (summation order only), stdError 1e-9 relative.
"""
import json
import os

import numpy as np
import pytest

import paper_2108_03076_b200 as E
from conftest import GOLD, load_kernel, load_model
from golden_util import ext_checksums
from oracle_py import Ref, ref_available

pytestmark = pytest.mark.gpu

PRICE_REL = 1e-13
SE_REL = 1e-9

BIG = json.load(open(os.path.join(GOLD, "big.json")))
KERN = {"brc": ("brc", "three"), "worst_off": ("worst-off", "three"),
        "call": ("european-call", "call")}


def ext_of(plan, kern, model, S):
    """Device spots [paths][steps][assets] in the reference's ext[rows][cols]
    layout (rowToDay / colToAsset, proj/src/pricing.cpp:182-198)."""
    L = plan.dump()
    order = model.get("order") or sorted(model["labels"])
    steps = [L["days"].index(d) for d in kern["rows"]]
    assets = [order.index(c) for c in kern["cols"]]
    return S[:, steps][:, :, assets]


@pytest.mark.parametrize("i", range(len(BIG["prices"])),
                         ids=[f'{p["name"]}-{p["paths"]}' for p in BIG["prices"]])
@pytest.mark.parametrize("jit", [False, True])
def test_headline_prices_match_reference(i, jit):
    p = BIG["prices"][i]
    kname, mname = KERN[p["name"]]
    res = E.price(load_kernel(kname), load_model(mname), p["paths"], p["seed"], p["days"],
                  jit=jit)
    for r, ph, sh in zip(res, p["price"], p["std_error"]):
        P, SE = float.fromhex(ph), float.fromhex(sh)
        assert abs(r["price"] - P) <= PRICE_REL * abs(P), (r["price"], P)
        assert abs(r["std_error"] - SE) <= SE_REL * SE, (r["std_error"], SE)


def test_brc_first_10k_paths_bit_exact():
    z = np.load(os.path.join(GOLD, "paths", "brc_10k.npz"))
    k, m = load_kernel("brc"), load_model("three")
    plan = E.Plan(E.Kernel(k), m, [0])
    n = len(z["payoffs"])
    sums, outs_all = [], []
    for p0 in range(0, n, 2500):
        outs, S, _, err = plan.debug_paths(int(z["seed"]), p0, 2500, spots=True)
        assert err == 2**64 - 1
        sums.append(ext_checksums(ext_of(plan, k, m, S)))
        outs_all.append(outs[:, 0])
    got = np.concatenate(sums)
    bad = np.flatnonzero(got != z["ext_checksum"])
    assert bad.size == 0, f"{bad.size} paths differ, first {bad[:5]}"
    pay = np.concatenate(outs_all)
    assert np.array_equal(pay, z["payoffs"]), int(np.sum(pay != z["payoffs"]))


@pytest.mark.skipif(not ref_available(), reason="oracle/_ref (compiled reference) absent")
@pytest.mark.parametrize("name,kern,model,n,days,seed", [
    ("brc", "brc", "three", 8_192, [0, 180], 1234),
    ("worst_off", "worst-off", "three", 200_000, [0, 150], 99),
    ("barrier", "barrier", "barrier", 100_000, [0, 5], 3)])
def test_per_path_payoffs_bit_exact_vs_compiled_reference(name, kern, model, n, days, seed):
    """The reference library itself (not the C restatement) evaluated on the
    box: every per-path payoff of the engine equals the reference's."""
    k, m = load_kernel(kern), load_model(model)
    for jit in (False, True):
        plan = E.Plan(E.Kernel(k), m, days, jit=jit)
        outs, _, _, err = plan.debug_paths(seed, 0, n)
        assert err == 2**64 - 1
        want = Ref().path_payoffs(k, m, seed, 0, n, days)
        assert np.array_equal(outs, want), (jit, int(np.sum(outs != want)))


@pytest.mark.skipif(not ref_available(), reason="oracle/_ref (compiled reference) absent")
def test_brc_price_vs_reference_run_on_the_box():
    """A fresh reference priceAcrossTime on the box's cores (not a fixture)."""
    k, m = load_kernel("brc"), load_model("three")
    want = Ref().price(k, m, 20_000, 2024, [0, 100], threads=os.cpu_count() or 1)
    got = E.price(k, m, 20_000, 2024, [0, 100])
    for g, w in zip(got, want):
        assert abs(g["price"] - w["price"]) <= PRICE_REL * abs(w["price"])
        assert abs(g["std_error"] - w["std_error"]) <= SE_REL * w["std_error"]
