"""The oracle (CPU restatement, oracle/cltk_oracle.c) pinned against the
reference: golden vectors generated from the compiled, unmodified reference
(oracle/make_golden.py) and, where it is built, the reference itself."""
import json
import math
import os

import numpy as np
import pytest

from conftest import GOLD, load_cases, load_kernel, load_model
from oracle_py import Oracle, OracleError, Ref, black_scholes_call, ref_available

ORACLE = Oracle()


def test_philox_random123_anchor():
    # Random123 philox2x64-10 KAT: ctr = key = 0 -> {ca00a0459843d731, 66c24222c9a845b5}
    assert ORACLE.philox_bits(0, 0, 0) == 0xca00a0459843d731 ^ 0x66c24222c9a845b5


def test_rng_kats_bit_exact():
    kat = json.load(open(os.path.join(GOLD, "rng_kat.json")))["kat"]
    for e in kat:
        assert ORACLE.philox_bits(e["seed"], e["path"], e["i"]) == int(e["bits"], 16)
        assert ORACLE.uniform(e["seed"], e["path"], e["i"]) == float.fromhex(e["uniform"])
        assert ORACLE.normal(e["seed"], e["path"], e["i"]) == float.fromhex(e["normal"])


def test_inverse_normal_bit_exact_and_domain():
    g = json.load(open(os.path.join(GOLD, "invnorm.json")))
    for e in g["inv"]:
        assert ORACLE.inv_normal_cdf(float.fromhex(e["p"])) == float.fromhex(e["x"])
    for e in g["cdf"]:
        assert ORACLE.normal_cdf(float.fromhex(e["x"])) == float.fromhex(e["cdf"])
    for p in g["domain_errors"]:
        with pytest.raises(OracleError):
            ORACLE.inv_normal_cdf(p)
    # proj/tests/test_pricing.cpp:40-50
    assert math.isclose(ORACLE.inv_normal_cdf(0.975), 1.959963984540054, rel_tol=1e-12)


def test_cholesky_known_factor_and_errors():
    # proj/tests/test_pricing.cpp:52-59
    l = ORACLE.cholesky([[1.0, 0.5], [0.5, 1.0]])
    assert l[0, 0] == 1.0 and l[1, 0] == 0.5 and math.isclose(l[1, 1], math.sqrt(0.75))
    with pytest.raises(OracleError):
        ORACLE.cholesky([[1.0, 2.0], [2.0, 1.0]])
    with pytest.raises(OracleError):
        ORACLE.cholesky([[1.0, 0.1], [0.2, 1.0]])


@pytest.mark.parametrize("case", [c["name"] for c in load_cases()])
def test_paths_and_payoffs_bit_exact(case):
    c = next(x for x in load_cases() if x["name"] == case)
    k, m = load_kernel(c["kernel"]), load_model(c["model"])
    z = np.load(os.path.join(GOLD, "paths", case + ".npz"))
    n = min(c["K"], 64)
    for p in range(n):
        assert np.array_equal(ORACLE.simulate_path(k, m, c["seed"], p), z["ext"][p])
        for d, day in enumerate(c["days"]):
            v = ORACLE.eval_kernel(k, z["ext"][p], z["disc"], day)
            assert v == z["payoffs"][p, d] or (math.isnan(v) and math.isnan(z["payoffs"][p, d]))


@pytest.mark.parametrize("case", [c["name"] for c in load_cases()])
def test_prices_bit_exact(case):
    c = next(x for x in load_cases() if x["name"] == case)
    k, m = load_kernel(c["kernel"]), load_model(c["model"])
    for pr in c["prices"]:
        if pr["paths"] > 200_000:
            continue
        res = ORACLE.price(k, m, pr["paths"], c["seed"], c["days"], threads=os.cpu_count() or 1)
        for r, p, s in zip(res, pr["price"], pr["std_error"]):
            assert r["price"] == float.fromhex(p)
            assert r["std_error"] == float.fromhex(s)


def test_black_scholes_constants():
    # proj/python/tests/test_smoke.py:51 and proj/tests/test_pricing.cpp:72-82
    assert math.isclose(black_scholes_call(100.0, 100.0, 0.05, 0.2, 90.0 / 365.0),
                        4.579032085233791, rel_tol=1e-12)
    assert math.isclose(black_scholes_call(100.0, 100.0, 0.0, 0.2, 90.0 / 365.0),
                        3.960376146988473, rel_tol=1e-9)


def test_eval_errors_match_reference_semantics():
    # kernel.cpp:207-211 division by zero; :186-193 type errors; :300-303 non-real result
    div = {"body": {"kind": "binop", "op": "div", "left": {"kind": "float", "value": 1.0},
                    "right": {"kind": "binop", "op": "sub",
                              "left": {"kind": "obsref", "row": 0, "col": 0},
                              "right": {"kind": "obsref", "row": 0, "col": 0}}},
           "rows": [5], "cols": ["A"], "tvars": [], "parties": [], "horizon": 6}
    with pytest.raises(OracleError, match="division by zero"):
        ORACLE.eval_kernel(div, np.array([[3.0]]), np.array([1.0]), 0)
    boolroot = {"body": {"kind": "bool", "value": True}, "rows": [], "cols": [], "tvars": [],
                "parties": [], "horizon": 1}
    with pytest.raises(OracleError, match="did not evaluate to a real"):
        ORACLE.eval_kernel(boolroot, np.zeros((0, 0)), np.zeros(0), 0)


@pytest.mark.skipif(not ref_available(), reason="oracle/_ref not built")
def test_reference_library_agrees_with_golden():
    ref = Ref()
    assert ref.philox_bits(0, 0, 0) == 0xacc2e26751eb9284
    c = next(x for x in load_cases() if x["name"] == "call")
    k, m = load_kernel("european-call"), load_model("call")
    r = ref.price(k, m, 1000, 42, [0], threads=2)
    assert r[0]["price"] == float.fromhex(c["prices"][1]["price"][0])


def test_restatement_pinned_on_the_first_brc_paths_of_the_big_fixture():
    """The C restatement against the reference's 10k-path BRC fixture
    (oracle/make_golden_big.py): ext checksums and payoffs of the first
    paths, and the 100k-path reference price."""
    from golden_util import ext_checksums
    z = np.load(os.path.join(GOLD, "paths", "brc_10k.npz"))
    k, m = load_kernel("brc"), load_model("three")
    n = 300
    ext = np.stack([ORACLE.simulate_path(k, m, 42, p) for p in range(n)])
    assert np.array_equal(ext_checksums(ext), z["ext_checksum"][:n])
    _, pay = ORACLE.price(k, m, n, 42, [0], threads=os.cpu_count() or 1, want_payoffs=True)
    assert np.array_equal(pay[0], z["payoffs"][:n])
    big = json.load(open(os.path.join(GOLD, "big.json")))
    p = next(x for x in big["prices"] if x["name"] == "brc" and x["paths"] == 100_000)
    r = ORACLE.price(k, m, 100_000, 42, [0], threads=os.cpu_count() or 1)[0]
    assert r["price"] == float.fromhex(p["price"][0])
    assert r["std_error"] == float.fromhex(p["std_error"][0])
