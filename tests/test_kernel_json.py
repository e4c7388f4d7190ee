"""Kernel JSON reader (csrc/host_model.cpp): the fast single-pass reader and
the DOM reader (nlohmann) produce the same kernel -- compared through the
compiled program listing of every golden kernel and variants with the
unusual cases (escapes fall back to the DOM path; malformed input raises
the DOM path's ContractParseError)."""
import json
import os

import pytest

import paper_2108_03076_b200 as E
from conftest import load_cases, load_kernel, load_model


def _listing(k, m, days, tenv=None):
    return E.compile_listing(E.Kernel(k), m, days, tenv=tenv)


def _both(k, m, days, tenv=None):
    fast = _listing(k, m, days, tenv)
    os.environ["CLTK_KERNEL_JSON_DOM"] = "1"
    try:
        dom = _listing(k, m, days, tenv)
    finally:
        del os.environ["CLTK_KERNEL_JSON_DOM"]
    return fast, dom


@pytest.mark.parametrize("case", load_cases(), ids=lambda c: c["name"])
def test_fast_reader_equals_dom_reader(case):
    k = json.dumps(load_kernel(case["kernel"]))
    fast, dom = _both(k, load_model(case["model"]), case["days"], case.get("tenv"))
    assert fast == dom


def test_text_forms_and_fallbacks():
    k = load_kernel("brc")
    m = load_model("three")
    pretty = json.dumps(k, indent=2)  # whitespace everywhere
    assert _both(pretty, m, [0])[0] == _listing(json.dumps(k), m, [0])
    esc = json.dumps(k).replace('"me"', '"m\\u0065"')  # an escape: DOM path, same kernel
    assert _listing(esc, m, [0]) == _listing(json.dumps(k), m, [0])
    for bad in ('{"body": {"kind": "float", "value": 1.0}', '{"body": 1}', '{not json'):
        with pytest.raises((E.ContractError, ValueError)):
            _listing(bad, m, [0])
