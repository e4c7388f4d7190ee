"""The host payoff compiler (csrc/compiler.cpp), checked on CPU: its program
listing, interpreted over the reference's own simulated spots, must
reproduce the reference evaluator's per-path payoffs BIT-FOR-BIT, for every
golden contract, every valuation day, with and without the min/max rewrite;
and its error channel must raise exactly where evalKernel raises."""
import json
import math
import os
import random

import numpy as np
import pytest

import paper_2108_03076_b200 as E
from conftest import GOLD, load_cases, load_kernel, load_model
from listing_interp import run_listing, spots_from_ext
from oracle_py import Oracle, OracleError, model_order

ORACLE = Oracle()


def same(a, b):
    a, b = np.asarray(a), np.asarray(b)
    return np.array_equal(a, b) or np.array_equal(np.isnan(a), np.isnan(b)) and np.array_equal(
        a[~np.isnan(a)], b[~np.isnan(b)])


@pytest.mark.parametrize("rewrite", [True, False])
@pytest.mark.parametrize("case", [c["name"] for c in load_cases()])
def test_listing_reproduces_reference_payoffs(case, rewrite):
    c = next(x for x in load_cases() if x["name"] == case)
    k, m = load_kernel(c["kernel"]), load_model(c["model"])
    L = E.compile_listing(E.Kernel(k), m, c["days"], tenv=c.get("tenv"), rewrite=rewrite)
    z = np.load(os.path.join(GOLD, "paths", case + ".npz"))
    S = spots_from_ext(L, k, model_order(m), z["ext"])
    vals, errs = run_listing(L, S, k)
    assert not errs.any()
    assert vals.shape == z["payoffs"].shape
    assert same(vals, z["payoffs"]), np.max(np.abs(vals - z["payoffs"]))


def test_brc_rewrite_streams_running_minima():
    k, m = load_kernel("brc"), load_model("three")
    L = E.compile_listing(E.Kernel(k), m, [0])
    ops = [o[0] for o in L["ops"]]
    # 1101 barrier tests -> 3 running minima updated once per simulated day
    assert ops.count("MIN") == 3 * 366
    assert ops.count("OR") < 10
    assert L["n_thread"] <= 16  # no materialised path
    L0 = E.compile_listing(E.Kernel(k), m, [0], rewrite=False)
    assert len(L0["ops"]) > 2 * len(L["ops"]) - 100


def test_step_schedule_is_streaming():
    # every op of a step only reads S-slots / registers / constants
    k, m = load_kernel("worst-off"), load_model("three")
    L = E.compile_listing(E.Kernel(k), m, [0])
    assert len(L["steps"]) == 5
    assert all(s["kind"] == 1 for s in L["steps"])  # all five days draw
    assert sum(s["end"] - s["begin"] for s in L["steps"]) == len(L["ops"])


def _random_kernel(rng: random.Random, depth: int, rows: int, cols: int, kind: str = "real"):
    """Random well- and ill-typed KExpr trees over ext/disc/t_now."""
    if depth == 0 or rng.random() < 0.2:
        if kind == "real":
            r = rng.random()
            if r < 0.45:
                return {"kind": "obsref", "row": rng.randrange(rows + 1), "col": rng.randrange(cols)}
            if r < 0.55:
                return {"kind": "payref", "row": rng.randrange(rows), "from": "you", "to": "me"}
            return {"kind": "float", "value": rng.choice([0.0, 1.0, 2.5, 100.0, -3.0, 0.5])}
        if kind == "bool":
            if rng.random() < 0.3:
                return {"kind": "bool", "value": rng.random() < 0.5}
            return {"kind": "binop", "op": "lt", "left": {"kind": "timeref", "row": rng.randrange(rows)},
                    "right": {"kind": "now"}}
        return {"kind": "nat", "value": rng.randrange(5)}
    if kind == "real":
        r = rng.random()
        if r < 0.6:
            op = rng.choice(["add", "sub", "mult", "div"])
            return {"kind": "binop", "op": op,
                    "left": _random_kernel(rng, depth - 1, rows, cols, "real"),
                    "right": _random_kernel(rng, depth - 1, rows, cols,
                                            "real" if rng.random() < 0.97 else "bool")}
        if r < 0.7:
            return {"kind": "unop", "op": "neg", "arg": _random_kernel(rng, depth - 1, rows, cols)}
        if r < 0.85:
            return {"kind": "if", "cond": _random_kernel(rng, depth - 1, rows, cols, "bool"),
                    "then": _random_kernel(rng, depth - 1, rows, cols),
                    "else": _random_kernel(rng, depth - 1, rows, cols)}
        return {"kind": "loopif", "window": rng.randrange(3),
                "cond": _random_kernel(rng, depth - 1, rows, cols, "bool"),
                "then": _random_kernel(rng, depth - 1, rows, cols),
                "else": _random_kernel(rng, depth - 1, rows, cols)}
    # bool
    r = rng.random()
    if r < 0.5:
        return {"kind": "binop", "op": rng.choice(["lt", "leq", "eq"]),
                "left": _random_kernel(rng, depth - 1, rows, cols),
                "right": _random_kernel(rng, depth - 1, rows, cols)}
    if r < 0.85:
        return {"kind": "binop", "op": rng.choice(["and", "or"]),
                "left": _random_kernel(rng, depth - 1, rows, cols, "bool"),
                "right": _random_kernel(rng, depth - 1, rows, cols, "bool")}
    return {"kind": "unop", "op": "not", "arg": _random_kernel(rng, depth - 1, rows, cols, "bool")}


def test_random_kernels_values_and_errors_match_reference_evaluator():
    """Differential test against the C restatement of evalKernel (itself
    pinned bit-exact to the reference): values, and the FIRST error in the
    reference's evaluation order (division by zero, out-of-range rows,
    type errors) -- including errors in untaken branches, which must NOT
    raise."""
    rng = random.Random(2108)
    model = {"rate": 0.01, "labels": {"A": {"spot": 1.0, "vol": 0.1}, "B": {"spot": 2.0, "vol": 0.1}}}
    n_checked = n_err = 0
    for trial in range(300):
        rows = rng.randrange(1, 4)
        body = _random_kernel(rng, 5, rows, 2)
        kern = {"body": body, "rows": sorted(rng.sample(range(1, 30), rows)), "cols": ["A", "B"],
                "tvars": [], "parties": ["you", "me"], "horizon": 31}
        days = [0, 5, 40]
        try:
            L = E.compile_listing(E.Kernel(kern), model, days)
        except E.ContractError as ex:  # statically unsupported shapes only
            assert ex.code == 4, ex
            continue
        K = 64
        ext = np.array([[[rng.choice([0.0, 1.0, 2.0, 2.5, -3.0, 100.0, rng.random()])
                          for _ in range(2)] for _ in range(rows)] for _ in range(K)])
        S = spots_from_ext(L, kern, ["A", "B"], ext)
        vals, errs = run_listing(L, S, kern)
        disc = np.array([math.exp(-0.01 * r / 365.0) for r in kern["rows"]])
        for p in range(K):
            for d, day in enumerate(days):
                try:
                    want = ORACLE.eval_kernel(kern, ext[p], disc, day)
                    want_err = None
                except OracleError as ex:
                    want_err = str(ex)
                site = int(errs[p, d])
                got_err = L["sites"][site][1] if site else None
                assert got_err == want_err, (trial, p, day, got_err, want_err)
                if want_err is None:
                    assert same(vals[p, d], want), (trial, p, day, vals[p, d], want)
                else:
                    n_err += 1
                n_checked += 1
    assert n_checked > 10000 and n_err > 100


def test_host_errors_match_reference_messages():
    call = E.Kernel(load_kernel("european-call"))
    m = load_model("call")
    with pytest.raises(E.ContractError, match="model has no asset spec for label AAPL") as ei:
        E.compile_listing(call, {"labels": {"MSFT": {"spot": 1.0, "vol": 0.1}}})
    assert ei.value.code == 5
    with pytest.raises(E.ContractError, match="not positive definite"):
        E.compile_listing(call, dict(m, corr=[[1.0, 2.0], [2.0, 1.0]],
                                     labels={"AAPL": m["labels"]["AAPL"],
                                             "B": {"spot": 1.0, "vol": 0.1}}))
    with pytest.raises(E.ContractError, match="size does not match"):
        E.compile_listing(call, dict(m, corr=[[1.0, 0.5], [0.5, 1.0]]))
    neg = {"body": {"kind": "obsref", "row": 0, "col": 0}, "rows": [-1], "cols": ["AAPL"],
           "tvars": [], "parties": [], "horizon": 0}
    with pytest.raises(E.ContractError, match="negative observation day"):
        E.compile_listing(E.Kernel(neg), m)
    tmpl = E.Kernel(load_kernel("template-option"))
    with pytest.raises(E.ContractError, match="unbound template variable: t0"):
        E.compile_listing(tmpl, m, tenv={})
    with pytest.raises(E.ContractParseError):
        E.compile_listing("{not json", m)


def test_batch_literal_pool_and_shape_check():
    brc = E.Kernel(load_kernel("brc"))
    m = load_model("three")
    inst = [brc.with_literals({2630.635: 3758.05 * f, 8288.0: 11840.0 * f, 840.0: 1200.0 * f})
            for f in (0.5, 0.6, 0.7, 0.8)]
    L = E.compile_listing(inst, m, [0])
    assert L["n_instances"] == 4 and L["n_inst_const"] == 3
    lo, hi = L["inst_code"]
    assert hi - lo <= 12  # per-instance work: 3 compares + a few boolean ops
    other = E.Kernel(load_kernel("worst-off"))
    with pytest.raises(E.ContractError, match="share one kernel shape"):
        E.compile_listing([brc, other], m, [0])


def test_template_literal_table_matches_instance_batch():
    brc = E.Kernel(load_kernel("brc"))
    lits = E.kernel_literals(brc)
    assert lits == brc.literals() and len(lits) == 1120
    m = load_model("three")
    fs = (0.5, 0.65, 0.8)
    inst = [brc.with_literals({2630.635: 3758.05 * f, 8288.0: 11840.0 * f, 840.0: 1200.0 * f})
            for f in fs]
    table = [k.literals() for k in inst]
    assert all(len(t) == 1120 for t in table)
    L1 = E.compile_listing(inst, m, [0])
    assert L1["n_inst_const"] == 3
    with pytest.raises(E.ContractError, match="literal table does not match"):
        E.Plan(brc, m, [0], literals=[lits[:-1]])


@pytest.mark.parametrize("name,model,tenv", [
    ("european-call", "call", None), ("barrier", "barrier", None),
    ("double-option", "double", None), ("fx-swap", "fx", None),
    ("template-option", "call", {"t0": 10, "t1": 80}), ("worst-off", "three", None),
    ("brc", "three", None)])
def test_kernel_text_format_compiles_like_json(name, model, tenv):
    """The reference's textual kernel format (emitKernelSource output, golden
    files written by the reference) is an engine input: same program as the
    kernel JSON, literal order included."""
    text = open(os.path.join(GOLD, "kernels", name + ".kernel")).read()
    js = load_kernel(name)
    m = load_model(model)
    days = [0, 10, 45]
    a = E.compile_listing(E.Kernel(js), m, days, tenv=tenv)
    b = E.compile_listing(text, m, days)
    for key in ("ops", "shared_const_bits", "outputs", "steps", "n_thread"):
        assert a[key] == b[key], key
    assert E.kernel_literals(text) == E.kernel_literals(E.Kernel(js))


def test_kernel_text_errors():
    with pytest.raises(E.ContractParseError, match="kernel source"):
        E.compile_listing("let rows = [1]\nlet cols = []\nlet payoffInternal(ext, tenv, disc, t0, t_now) = (1.0 +",
                          load_model("call"))
