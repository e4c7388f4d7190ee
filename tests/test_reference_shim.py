"""The reference-side binding (integration/cltk_reference_shim.cpp), compiled
against the reference's own headers and linked next to the unmodified
reference library (oracle/_ref/libcltk_shim.so, built by oracle/Makefile).

The chain is the reference's own `cltk price` flow (proj/tools/cli.cpp:246-259):
parseContract -> typeCheckContr -> compileContract -> cutPayoff -> reindex
(all reference code) -> cltk::gpu::priceAcrossTime (the shim: kernelToJson /
tenvToJson / the ModelSpec writer -> cltk_gpu_price) -- compared with the
reference's CPU cltk::priceAcrossTime / priceMC on the same cltk::Kernel.
The five shipped contracts start from their IL wire format (the repo does not
copy the reference's contract sources), the BASELINE contracts from CL text.
"""
import ctypes as C
import json
import os

import numpy as np
import pytest

from conftest import GOLD, ROOT, load_model

pytestmark = pytest.mark.gpu

SHIM = os.path.join(ROOT, "oracle", "_ref", "libcltk_shim.so")
PRICE_REL = 1e-13
SE_REL = 1e-9


@pytest.fixture(scope="module")
def shim():
    if not os.path.exists(SHIM):
        pytest.skip("oracle/_ref/libcltk_shim.so not built (needs the reference headers)")
    L = C.CDLL(SHIM)
    u64, dbl = C.c_uint64, C.c_double
    L.cltkshim_last_error.restype = C.c_char_p
    L.cltkshim_price.restype = C.c_int
    L.cltkshim_price.argtypes = [C.c_char_p, C.c_int, C.c_char_p, C.c_char_p, u64, u64,
                                 C.c_void_p, C.c_size_t, C.c_int, C.c_uint, C.c_void_p,
                                 C.c_void_p]
    L.cltkshim_price_mc.restype = C.c_int
    L.cltkshim_price_mc.argtypes = [C.c_char_p, C.c_char_p, u64, u64, u64, C.c_int,
                                    C.POINTER(dbl), C.POINTER(dbl)]
    return L


def _price(L, src, kind, tenv, model, paths, seed, days, engine):
    d = np.ascontiguousarray(days, dtype=np.uint64)
    p = np.zeros(len(d))
    s = np.zeros(len(d))
    rc = L.cltkshim_price(src.encode(), kind, json.dumps(tenv or {}).encode(),
                          json.dumps(model).encode(), paths, seed, d.ctypes.data, len(d),
                          engine, os.cpu_count() or 1, p.ctypes.data, s.ctypes.data)
    return rc, L.cltkshim_last_error().decode(), p, s


CASES = [  # (source, kind, tenv, model, paths, seed, days)
    ("il/european-call_nocut.json", 1, {}, "call", 200_000, 42, [0, 45, 91]),
    ("il/barrier_nocut.json", 1, {}, "barrier", 50_000, 11, [0, 10]),
    ("il/double-option_nocut.json", 1, {}, "double", 50_000, 3, [0, 30, 45]),
    ("il/fx-swap_nocut.json", 1, {}, "fx", 20_000, 1, [0, 30, 60, 90]),
    ("il/template-option_nocut_t1.json", 1, None, "call", 20_000, 9, [0, 10, 50, 91]),
    ("contracts/worst-off.cl", 0, {}, "three", 400_000, 42, [0, 100]),
    ("contracts/brc.cl", 0, {}, "three", 20_000, 42, [0, 180]),
]


def _source(rel):
    if rel.startswith("contracts/"):
        return open(os.path.join(ROOT, rel)).read(), None
    obj = json.load(open(os.path.join(GOLD, rel)))
    return json.dumps(obj["il"]), obj.get("tenv")


@pytest.mark.parametrize("rel,kind,tenv,model,paths,seed,days", CASES, ids=[c[0] for c in CASES])
def test_shim_matches_reference_price_across_time(shim, rel, kind, tenv, model, paths, seed,
                                                  days):
    src, fixture_tenv = _source(rel)
    tenv = fixture_tenv if tenv is None else tenv
    m = load_model(model)
    rc0, e0, p0, s0 = _price(shim, src, kind, tenv, m, paths, seed, days, engine=0)
    rc1, e1, p1, s1 = _price(shim, src, kind, tenv, m, paths, seed, days, engine=1)
    assert rc0 == 0, e0
    assert rc1 == 0, e1
    assert np.all(np.abs(p1 - p0) <= PRICE_REL * np.abs(p0) + 1e-300), (p1, p0)
    assert np.all(np.abs(s1 - s0) <= SE_REL * s0 + 1e-14 * np.abs(p0)), (s1, s0)


def test_shim_price_mc_and_errors_match_reference(shim):
    src = open(os.path.join(ROOT, "contracts", "worst-off.cl")).read()
    m = load_model("three")
    out = []
    for engine in (0, 1):
        p, s = C.c_double(), C.c_double()
        rc = shim.cltkshim_price_mc(src.encode(), json.dumps(m).encode(), 100_000, 7, 73,
                                    engine, C.byref(p), C.byref(s))
        assert rc == 0, shim.cltkshim_last_error()
        out.append((p.value, s.value))
    assert abs(out[1][0] - out[0][0]) <= PRICE_REL * abs(out[0][0])
    # the reference's errors cross the shim with the reference's code and text
    for model, paths in (({"rate": 0.03, "labels": {"SX5E": {"spot": 1.0, "vol": 0.1}}}, 1000),
                         (m, 0)):
        got = []
        for engine in (0, 1):
            rc, msg, _, _ = _price(shim, src, 0, {}, model, paths, 1, [0], engine)
            got.append((rc, msg))
        assert got[0][0] == 5 and got[0] == got[1], got
