"""NVRTC payoff kernels (csrc/jit.cpp): the compiled payoff program emitted as
CUDA and built for sm_100a at plan creation.

CPU: every golden contract's generated source NVRTC-compiles for sm_100a (no
device needed) and the generator's structure (step classes, spots from
registers, literals as kernel data).
GPU: prices through the NVRTC kernel equal the interpreter's bit for bit --
same ops, same order, same IEEE operations -- for every golden case, both RNG
modes, template batches and literal tables, and the error channel.
"""
import os
import re

import numpy as np
import pytest

import paper_2108_03076_b200 as E
from conftest import load_cases, load_kernel, load_model

CASES = load_cases()


def _case(name):
    return next(x for x in CASES if x["name"] == name)


@pytest.mark.parametrize("kern,model,days,tenv", [
    ("european-call", "call", [0, 45], {}),
    ("barrier", "barrier", [0, 10], {}),
    ("double-option", "double", [0, 30, 45], {}),
    ("fx-swap", "fx", [0, 30, 60, 90], {}),
    ("template-option", "call", [0, 10, 50], {"t0": 10, "t1": 80}),
    ("worst-off", "three", [0, 100], {}),
    ("brc", "three", [0, 180], {}),
])
def test_generated_source_compiles_for_sm100a(kern, model, days, tenv):
    src = E.jit_source(E.Kernel(load_kernel(kern)), load_model(model), days, tenv)
    assert "cltk_jit_path" in src and "path_body<" in src
    n, log = E.jit_compile(src)
    assert n > 0, log


def test_brc_source_structure():
    """BRC 3 x 367: 365 identical running-min steps share one class; the spots
    are read from registers; the barrier/strike literals are table operands
    (JC), never baked in (new literal values reuse the compiled kernel)."""
    k = E.Kernel(load_kernel("brc"))
    m = load_model("three")
    src = E.jit_source(k, m, [0])
    cases = re.findall(r"case (\d+): \{", src)
    assert len(cases) == 3, cases
    # spots arrive as logarithms; the running minima stay in the log domain
    # (log_fmin_b: the range-checked form is dropped when the host bounds the log-spots)
    assert "kLogSpots = true" in src and "L[0]" in src and ("log_fmin(" in src or "log_fmin_b(" in src)
    for lit in ("2630.635", "8288", "840"):
        assert lit not in src
    # a different literal instance of the template: identical source
    lo = k.with_literals({2630.635: 1879.0, 8288.0: 5920.0, 840.0: 600.0})
    assert E.jit_source(lo, m, [0]) == src
    sobol = E.jit_source(k, m, [0], rng="sobol")
    assert "path_body<3, true" in sobol and "path_body<3, false" in src


def test_jit_modes_validated():
    with pytest.raises(ValueError):
        E.price(E.Kernel(load_kernel("european-call")), load_model("call"), 10, 1, jit="yes")


def _bits(rs):
    return [(float(r["price"]).hex(), float(r["std_error"]).hex()) for r in rs]


@pytest.mark.gpu
@pytest.mark.parametrize("case", [c["name"] for c in CASES])
def test_jit_prices_equal_interpreter_bitwise(case):
    c = _case(case)
    k, m = E.Kernel(load_kernel(c["kernel"])), load_model(c["model"])
    n = 50_000 if c["kernel"] != "brc" else 20_000
    a = E.price(k, m, n, c["seed"], c["days"], c["tenv"])
    b = E.price(k, m, n, c["seed"], c["days"], c["tenv"], jit=True)
    assert _bits(a) == _bits(b)


@pytest.mark.gpu
def test_jit_plan_reports_nvrtc_and_matches_reference_case():
    c = _case("worst_off_days")
    k, m = E.Kernel(load_kernel(c["kernel"])), load_model(c["model"])
    plan = E.Plan(k, m, c["days"], jit=True)
    assert plan.info["jit"] == 1
    assert E.Plan(k, m, c["days"]).info["jit"] == 0
    assert E.Plan(k, m, c["days"], jit="auto").info["jit"] == 1
    # the reference's own prices at the golden path counts (summation order only)
    for pr in c["prices"]:
        got = E.price(k, m, pr["paths"], c["seed"], c["days"], jit=True)
        for g, p in zip(got, pr["price"]):
            P = float.fromhex(p)
            assert abs(g["price"] - P) <= 1e-13 * abs(P) + 1e-13, (g["price"], P)


@pytest.mark.gpu
@pytest.mark.parametrize("kern,model", [("brc", "three"), ("worst-off", "three"),
                                        ("european-call", "call")])
def test_jit_qmc_equals_interpreter_bitwise(kern, model):
    k, m = E.Kernel(load_kernel(kern)), load_model(model)
    a = E.price(k, m, 40_000, 3, [0], rng="sobol")
    b = E.price(k, m, 40_000, 3, [0], rng="sobol", jit=True)
    assert _bits(a) == _bits(b)


@pytest.mark.gpu
def test_jit_template_batch_and_literal_table_bitwise():
    brc = E.Kernel(load_kernel("brc"))
    m = load_model("three")
    insts = [brc.with_literals({2630.635: 3758.05 * f, 8288.0: 11840.0 * f, 840.0: 1200.0 * f})
             for f in (0.5, 0.7, 0.9)]
    a = E.price_batch(insts, m, 20_000, 42)
    b = E.price_batch(insts, m, 20_000, 42, jit=True)
    assert [_bits(x) for x in a] == [_bits(x) for x in b]
    lits = np.array([E.kernel_literals(x) for x in insts])
    c = E.price_template(brc, lits, m, 20_000, 42, jit=True)
    assert [_bits(x) for x in c] == [_bits(x) for x in a]


@pytest.mark.gpu
def test_jit_division_by_zero_raises_like_interpreter():
    kern = {"body": {"kind": "binop", "op": "div", "left": {"kind": "float", "value": 1.0},
                     "right": {"kind": "binop", "op": "sub",
                               "left": {"kind": "obsref", "row": 0, "col": 0},
                               "right": {"kind": "obsref", "row": 0, "col": 0}}},
            "rows": [5], "cols": ["AAPL"], "tvars": [], "parties": [], "horizon": 6}
    with pytest.raises(E.ContractError, match="kernel: division by zero") as ei:
        E.price(E.Kernel(kern), load_model("call"), 1000, 1, jit=True)
    assert ei.value.code == 5
    safe = {"body": {"kind": "if", "cond": {"kind": "bool", "value": False},
                     "then": kern["body"], "else": {"kind": "float", "value": 2.0}},
            "rows": [5], "cols": ["AAPL"], "tvars": [], "parties": [], "horizon": 6}
    assert E.price(E.Kernel(safe), load_model("call"), 1000, 1, jit=True)[0]["price"] == 2.0


def _up_barrier_brc():
    """The BRC with its knock-in turned into an up-and-in at 130% of spot
    (literal on the left of <=): the OR chains become running maxima."""
    k = load_kernel("brc")
    up = {2630.635: 3758.05 * 1.3, 8288.0: 11840.0 * 1.3, 840.0: 1200.0 * 1.3}

    def walk(e):
        if isinstance(e, dict):
            if (e.get("kind") == "binop" and e.get("op") == "leq" and
                    e["left"].get("kind") == "obsref" and e["right"].get("kind") == "float" and
                    e["right"]["value"] in up):
                return {"kind": "binop", "op": "leq",
                        "left": {"kind": "float", "value": up[e["right"]["value"]]},
                        "right": e["left"]}
            return {kk: walk(v) for kk, v in e.items()}
        if isinstance(e, list):
            return [walk(v) for v in e]
        return e
    return walk(k)


def test_up_barrier_source_uses_log_fmax():
    src = E.jit_source(E.Kernel(_up_barrier_brc()), load_model("three"), [0, 100])
    assert ("log_fmax(" in src or "log_fmax_b(" in src) and "kLogSpots = true" in src


def test_qmc_log_spots_bounded_by_the_bridge():
    """QMC plans get the range-check-free log-domain ops too: the host bounds
    every log-spot by running the bridge program on |W| bounds (AS241 of
    32-bit Sobol points: |z| < 6.5)."""
    src = E.jit_source(E.Kernel(load_kernel("brc")), load_model("three"), [0], rng="sobol")
    assert "log_fmin_b(" in src and "log_fmin(" not in src
    # a model whose log-spots can leave (-500, 500) keeps the checked forms
    import copy
    wild = copy.deepcopy(load_model("three"))
    for v in wild["labels"].values():
        v["vol"] = 40.0
    src = E.jit_source(E.Kernel(load_kernel("brc")), wild, [0], rng="sobol")
    assert "log_fmin(" in src and "log_fmin_b(" not in src


def _brc_batch_literals(n=64):
    """n instances of the BRC template: knock-in barrier 50..80 % of spot,
    strike (initial fixing) 90..110 % of spot."""
    import numpy as np
    kj = load_kernel("brc")
    base = E.kernel_literals(kj)
    spots = {3758.05: 2630.635, 11840.0: 8288.0, 1200.0: 840.0}
    rows = []
    for i in range(n):
        b = 0.5 + 0.3 * i / (n - 1)
        r = 0.9 + 0.2 * ((i * 7) % n) / (n - 1)
        sub = {bar: sp * b for sp, bar in spots.items()}
        sub.update({sp: sp * r for sp in spots})
        rows.append([sub.get(v, v) for v in base])
    return kj, np.asarray(rows)


def test_template_batch_minima_stay_log_domain_until_the_last_step():
    """C4 BRC batch: the knock-in minima are compared with per-instance
    barriers in the instance section, so they must reach it as spots.  They
    stay logarithms through the 365 running-minimum steps (log_fmin, no exp
    per step) and the last step exponentiates each one once."""
    kj, lit = _brc_batch_literals()
    src = E.jit_source(E.Kernel(kj), load_model("three"), [0], literals=lit)
    cases = re.split(r"case \d+: \{", src.split("static __device__ __forceinline__ void inst(")[0])[1:]
    assert len(cases) == 3
    mins = [c for c in cases if "log_fmin" in c]
    assert len(mins) == 2, "running-min classes in the log domain"
    running, last = (mins[0], mins[1]) if mins[0].count("spot_exp") < mins[1].count("spot_exp") else (mins[1], mins[0])
    assert "spot_exp" not in running  # 365 steps without an exp
    assert last.count("spot_exp") == 6  # three minima + the three final spots, once each


def test_template_batch_divides_by_host_reciprocals():
    """The instance-major section divides each spot by the instance's literal
    through RN(1/literal) from extra literal columns (3 FP64 operations,
    Markstein's exact rounding) -- only while every instance value of that
    literal lies in [2^-100, 2^100]; otherwise the full IEEE division stays."""
    kj, lit = _brc_batch_literals()
    m = load_model("three")
    src = E.jit_source(E.Kernel(kj), m, [0], literals=lit)
    inst_t = src.split("inst_t(")[1]
    assert inst_t.count("div_recip(") == 3 and "__ddiv_rn" not in inst_t
    recip = [int(c) for c in re.findall(r"div_recip\(a, b, JI\((\d+)\)\)", inst_t)]
    plain = [int(c) for c in re.findall(r"= JI\((\d+)\);", src)]
    assert len(set(recip)) == 3 and min(recip) > max(plain)  # appended columns
    bad = lit.copy()
    base = list(E.kernel_literals(kj))
    for c, v in enumerate(base):  # one instance's first-asset fixing out of range
        if v == 3758.05:
            bad[5, c] = 1e-40  # below 2^-100
    src = E.jit_source(E.Kernel(kj), m, [0], literals=bad)
    inst_t = src.split("inst_t(")[1]
    assert inst_t.count("div_recip(") == 2 and inst_t.count("__ddiv_rn") == 1


def test_step_divisions_by_shared_constants_use_reciprocals():
    """The worst-off's per-step performance ratios (spot / initial fixing, a
    shared literal) divide through RN(1/fixing) appended to the shared
    constants: 15 div_recip per path, no IEEE division left; a fixing out of
    [2^-100, 2^100] keeps the IEEE division for that operand."""
    k = load_kernel("worst-off")
    m = load_model("three")
    src = E.jit_source(E.Kernel(k), m, [0])
    assert src.count("div_recip(") == 15 and "__ddiv_rn" not in src
    base = E.kernel_literals(k)
    tiny = E.Kernel(k).with_literals({3758.05: 1e-40}) if 3758.05 in base else None
    if tiny is not None:
        src = E.jit_source(tiny, m, [0])
        assert "__ddiv_rn" in src


@pytest.mark.gpu
def test_template_batch_log_domain_minima_bitwise():
    """The same batch priced with the NVRTC kernel (log-domain minima,
    exponentiated at the last step) and the interpreter (spot-domain minima):
    bit-identical instance prices."""
    kj, lit = _brc_batch_literals(40)
    m = load_model("three")
    a = E.price_template(kj, lit, m, 30000, 11, jit=False)
    b = E.price_template(kj, lit, m, 30000, 11, jit=True)
    assert len(a) == len(b) == 40
    for ra, rb in zip(a, b):
        x, y = ra[0], rb[0]
        assert x["price"] == y["price"] and x["std_error"] == y["std_error"], (x, y)


@pytest.mark.gpu
@pytest.mark.parametrize("variant", ["down", "up"])
def test_log_domain_extrema_bitwise_vs_interpreter(variant):
    """Log-domain running minima (BRC knock-in) and maxima (up-and-in
    variant): NVRTC prices equal the interpreter's bit for bit, several
    valuation days, both RNG modes."""
    k = E.Kernel(load_kernel("brc") if variant == "down" else _up_barrier_brc())
    m = load_model("three")
    for rng in ("philox", "sobol"):
        a = E.price(k, m, 40000, 7, [0, 100, 300], rng=rng, jit=False)
        b = E.price(k, m, 40000, 7, [0, 100, 300], rng=rng, jit=True)
        for x, y in zip(a, b):
            assert x["price"] == y["price"] and x["std_error"] == y["std_error"], (rng, x, y)


@pytest.mark.gpu
@pytest.mark.parametrize("kern,model,days,paths", [("worst-off", "three", [0, 100, 300], 1 << 20),
                                                   ("european-call", "call", [0, 30, 60],
                                                    (1 << 22) + 64)])
def test_qmc_multi_day_reduction_deterministic(kern, model, days, paths):
    """Regression: QMC plans with several outputs park the per-path values
    in the normal scratch.  Parked in rows counted from X they once landed in
    other threads' data -- behind a half-row P region in other threads'
    bridge slots (odd batch sizes, the worst-off), and inside P itself, whose
    32-bit Sobol integers pack two threads per double (one-asset models, the
    call) -- races that changed random chunks of multi-day QMC prices from
    launch to launch.  QMC now parks in its bridge-slot rows.  Repeated
    launches must give one bit pattern, the interpreter's."""
    from paper_2108_03076_b200.distributed import DistributedPricer
    import torch
    m = load_model(model)
    stream = torch.cuda.current_stream(0).cuda_stream
    ref = None
    for jit in (False, True):
        pr = DistributedPricer(E.Kernel(load_kernel(kern)), m, days, device=0,
                               rng="sobol", jit=jit)
        _, nc = pr.plan.chunking(paths)
        for _ in range(12 if jit else 4):
            parts = pr.partials(paths)
            parts.zero_()
            pr.plan.launch(paths, 20, 0, nc, parts.data_ptr(), stream)
            torch.cuda.synchronize()
            bits = parts.view(torch.int64).clone()
            if ref is None:
                ref = bits
            assert torch.equal(bits, ref)


@pytest.mark.gpu
def test_disk_cache_reuses_and_repairs_the_cubin(tmp_path):
    """The NVRTC cubin of a program is written to CLTK_JIT_CACHE_DIR and loaded
    by a later process; a damaged entry is recompiled, never trusted."""
    import subprocess
    import sys
    code = ("import sys; sys.setrecursionlimit(100000); import paper_2108_03076_b200 as E, json;"
            "from conftest import load_kernel, load_model;"
            "r = E.price(E.Kernel(load_kernel('worst-off')), load_model('three'), 4096, 5, jit=True);"
            "print(json.dumps(r[0]['price'].hex()))")
    env = dict(os.environ, CLTK_JIT_CACHE_DIR=str(tmp_path))
    here = os.path.dirname(os.path.abspath(__file__))
    env["PYTHONPATH"] = os.pathsep.join([os.path.dirname(here), here, env.get("PYTHONPATH", "")])
    run = lambda: subprocess.run([sys.executable, "-c", code], env=env, capture_output=True,
                                 text=True, timeout=300)
    a = run()
    assert a.returncode == 0, a.stderr
    files = list(tmp_path.glob("*.cubin"))
    assert len(files) == 1 and files[0].stat().st_size > 0
    b = run()
    assert b.returncode == 0 and b.stdout == a.stdout
    files[0].write_bytes(b"not a cubin")
    c = run()
    assert c.returncode == 0 and c.stdout == a.stdout, c.stderr
    assert files[0].read_bytes() != b"not a cubin"
