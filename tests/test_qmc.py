"""QMC mode (Sobol + AS241 + Brownian bridge), CPU checks.  The reference
has no QMC; these pin the mode to third-party references:
scipy's Sobol integers and ndtri, and the bridge's defining covariance."""
import os

import numpy as np
import pytest

import paper_2108_03076_b200 as E
from conftest import GOLD, ROOT, load_kernel, load_model
from qmc_oracle import (as241, bridge_nodes, bridge_paths, load_direction_numbers,
                        sobol_int)

TABLE = os.path.join(ROOT, "paper_2108_03076_b200", "csrc", "sobol_table.cpp")


def test_as241_matches_scipy_ndtri():
    sp = pytest.importorskip("scipy.special")
    rng = np.random.default_rng(3)
    p = np.concatenate([rng.random(200_000), 10 ** -rng.uniform(3, 300, 20_000),
                        1 - 10 ** -rng.uniform(3, 15, 20_000)])
    x, y = as241(p), sp.ndtri(p)
    assert np.max(np.abs(x - y) / np.maximum(np.abs(y), 1e-300)) < 2e-15


def test_shipped_direction_numbers_reproduce_scipy_sobol():
    qmc = pytest.importorskip("scipy.stats.qmc")
    v = load_direction_numbers(TABLE)
    assert v.shape == (2048, 32)
    dims = [0, 1, 2, 7, 100, 1097, 2047]
    pts = (qmc.Sobol(d=2048, scramble=False, bits=32).random(1024) * 2.0**32).astype(np.uint64)
    x = sobol_int(v, dims, np.arange(1024))
    assert np.array_equal(x.astype(np.uint64), pts[:, dims])


def test_bridge_schedule_reproduces_direct_bridge():
    """Run the engine's compiled bridge program (pre-order computes into
    slots, in-order emits) in numpy and compare with the direct construction."""
    k, m = load_kernel("brc"), load_model("three")
    L = E.compile_listing(E.Kernel(k), m, [0], rng="sobol")
    steps = [s for s in L["steps"] if s["kind"] == 1]
    nD, nA = len(steps), L["n_assets"]
    tau = np.array([d for d, s in zip(L["days"], L["steps"]) if s["kind"] == 1]) / 365.0
    rng = np.random.default_rng(5)
    K = 16
    Z = rng.standard_normal((K, nD, nA))  # node-indexed
    Wd = bridge_paths(tau, Z)
    slots = np.zeros((L["bridge_slots"], K, nA))
    got = np.zeros((K, nD, nA))
    for si, s in enumerate(steps):
        b0, b1, e = s["br"]
        for (node, dst, l, r, wl, wr, sd) in L["bridge"][b0:b1]:
            Wl = 0.0 if l < 0 else slots[l]
            Wr = 0.0 if r < 0 else slots[r]
            slots[dst] = wl * Wl + wr * Wr + sd * Z[:, node]
        got[:, si] = slots[e]
    np.testing.assert_allclose(got, Wd, rtol=1e-12, atol=1e-12)
    assert L["bridge_slots"] <= 2 + int(np.ceil(np.log2(nD))) + 1
    # every node exactly once, BFS node 0 = terminal point
    assert sorted(b[0] for b in L["bridge"]) == list(range(nD))


def test_bridge_covariance_is_min_s_t():
    tau = np.array([0.1, 0.25, 0.3, 0.7, 1.0, 1.3])
    rng = np.random.default_rng(0)
    W = bridge_paths(tau, rng.standard_normal((400_000, len(tau), 1)))[:, :, 0]
    C = np.cov(W.T)
    np.testing.assert_allclose(C, np.minimum.outer(tau, tau), atol=0.01)


def test_sobol_mode_limits():
    k = E.Kernel(load_kernel("brc"))
    big = {"rate": 0.0, "labels": {l: {"spot": 1.0, "vol": 0.1} for l in
                                   ["SX5E", "N225", "SPX", "A", "B", "C", "D"]},
           "order": ["SX5E", "N225", "SPX", "A", "B", "C", "D"]}
    with pytest.raises(E.ContractError, match="Sobol mode supports at most 2048"):
        E.compile_listing(k, big, [0], rng="sobol")
