"""reindex: the engine's IL -> kernel producer
(csrc/reindex.cpp, restating proj/src/kernel.cpp:14-180) against the
reference's own reindex output for every golden contract, before and after
cutPayoff and under several template environments (tests/golden/il/, made by
oracle/make_golden_il.py from the compiled reference).  Host only.
GPU: a reindexed kernel prices bit-identically to the reference's kernel."""
import copy
import glob
import json
import os

import pytest

import paper_2108_03076_b200 as E
from conftest import GOLD, load_kernel, load_model

IL_CASES = sorted(glob.glob(os.path.join(GOLD, "il", "*.json")))


def _load(path):
    with open(path) as f:
        return json.load(f)


@pytest.mark.parametrize("path", IL_CASES, ids=[os.path.basename(p)[:-5] for p in IL_CASES])
def test_reindex_matches_reference(path):
    g = _load(path)
    k = E.reindex(g["il"], g["tenv"])
    assert json.loads(k.json) == g["kernel"]


def test_cut_il_gives_the_golden_pricing_kernels():
    """reindex(cutPayoff(IL)) is exactly the kernel the pricing fixtures use."""
    for name in ("european-call", "barrier", "double-option", "fx-swap", "worst-off", "brc"):
        g = _load(os.path.join(GOLD, "il", name + ".json"))
        assert json.loads(E.reindex(g["il"], g["tenv"]).json) == load_kernel(name)


def test_reindex_errors_like_the_reference():
    g = _load(os.path.join(GOLD, "il", "template-option.json"))
    with pytest.raises(E.ContractError) as ei:  # UnboundTemplateVar is an EvalError
        E.reindex(g["il"], {})
    assert "unbound template variable" in str(ei.value)
    bad = copy.deepcopy(g["il"])
    bad["kind"] = "nonsense"
    with pytest.raises(E.ContractParseError):
        E.reindex(bad, g["tenv"])
    with pytest.raises(E.ContractParseError):
        E.reindex("{not json", g["tenv"])


def test_window_variable_round_trips_through_the_kernel_json():
    """A LoopIf window bound from a template variable is materialised with
    its slack rows and keeps its windowVar (kernel.cpp:160-168, :565)."""
    il = {"kind": "loopif", "window": {"kind": "tvar", "name": "w"},
          "cond": {"kind": "binop", "op": "leq",
                   "left": {"kind": "model", "label": "A", "time": {"kind": "tnumz", "value": 0}},
                   "right": {"kind": "float", "value": 90.0}},
          "then": {"kind": "payoff", "time": {"kind": "texpr", "value": {"kind": "tnum", "value": 0}},
                   "from": "you", "to": "me"},
          "else": {"kind": "float", "value": 0.0}}
    k = json.loads(E.reindex(il, {"w": 3}).json)
    assert k["body"]["window"] == 3 and k["body"]["windowVar"] == 0 and k["tvars"] == ["w"]
    assert k["rows"] == [0, 1, 2, 3] and k["horizon"] == 4 and k["parties"] == ["you", "me"]


@pytest.mark.gpu
def test_reindexed_kernel_prices_like_the_reference_kernel():
    g = _load(os.path.join(GOLD, "il", "worst-off.json"))
    m = load_model("three")
    a = E.price(E.reindex(g["il"], g["tenv"]), m, 50_000, 42, [0, 100])
    b = E.price(E.Kernel(load_kernel("worst-off")), m, 50_000, 42, [0, 100])
    assert a == b
