"""The engine's restatements of glibc exp / log / erfc (csrc/glibc_math.h,
host build) are bit-identical to the system libm the reference links --
the precondition for bit-exact normals and spots on the device."""
import ctypes as C
import os
import subprocess

import numpy as np
import pytest

from conftest import ROOT

LIB = os.path.join(ROOT, "build", "libgm_check.so")


@pytest.fixture(scope="module")
def gm():
    subprocess.run(["make", "-C", ROOT, "-s", "testlib"], check=True)
    L = C.CDLL(LIB)
    L.gm_check.restype = C.c_long
    L.gm_check.argtypes = [C.c_int, C.c_void_p, C.c_long, C.POINTER(C.c_long)]
    return L


def check(L, fn, xs):
    xs = np.ascontiguousarray(xs, dtype=np.float64)
    first = C.c_long()
    bad = L.gm_check(fn, xs.ctypes.data, len(xs), C.byref(first))
    assert bad == 0, (bad, xs[first.value] if first.value >= 0 else None)


def test_exp_bit_exact(gm):
    rng = np.random.default_rng(11)
    check(gm, 0, rng.uniform(0.0, 40.0, 400_000))          # Halley's exp(x*x/2)
    check(gm, 0, rng.uniform(2.0, 12.0, 400_000))          # spots exp(logS)
    check(gm, 0, rng.uniform(-745.0, 709.0, 200_000))
    check(gm, 0, np.concatenate([rng.uniform(-1e-14, 1e-14, 1000), rng.uniform(-760, -700, 5000),
                                 [0.0, -0.0, 709.78, -745.13, 800.0, -800.0, np.inf, -np.inf,
                                  np.nan]]))


def test_log_bit_exact(gm):
    rng = np.random.default_rng(12)
    check(gm, 1, rng.uniform(2.0**-54, 0.02425, 400_000))  # invNormalCdf tails
    check(gm, 1, np.exp(rng.uniform(-745, 709, 200_000)))
    check(gm, 1, rng.uniform(0.93, 1.07, 200_000))         # near-1 path
    check(gm, 1, [5e-324, 1e-310, 2.2e-308, 0.0, -0.0, -1.0, np.inf, np.nan, 1.0])


def test_erfc_bit_exact(gm):
    rng = np.random.default_rng(13)
    check(gm, 2, rng.uniform(-6.0, 6.0, 600_000))          # Halley's erfc(-x/sqrt 2)
    check(gm, 2, rng.uniform(-30.0, 30.0, 100_000))
    edges = [0.84375, 1.25, 1 / 0.35, 6.0, 28.0, 2.0**-56, 0.25]
    pts = []
    for e in edges:
        for s in (1, -1):
            pts += list(np.nextafter(s * e, [-np.inf, np.inf])) + [s * e]
    check(gm, 2, pts + [0.0, -0.0, np.inf, -np.inf, np.nan])
