"""Test helper: vectorised numpy interpreter of the engine's compiled program
listing (``compile_listing``), fed with the reference's own simulated spots.

It lets the CPU suite check the payoff COMPILER bit-for-bit against the
reference evaluator (golden per-path payoffs from evalKernel) without a GPU.
It is a checker of the compiler's output, never part of the pricing path.
"""
from __future__ import annotations

import numpy as np

NAN = np.float64("nan")


def run_listing(L: dict, S: np.ndarray, kernel: dict) -> tuple[np.ndarray, np.ndarray]:
    """S: [K][n_steps][n_assets] spots (only observed entries are read).
    Returns (values [K][n_out], error-site [K][n_out])."""
    K = S.shape[0]
    nA, nT = L["n_assets"], L["n_thread"]
    nS, nI = L["n_shared_const"], L["n_inst_const"]
    sc = np.array(L["shared_const_bits"], dtype=np.uint64).view(np.float64)
    inst = np.array(L["inst_const"], dtype=np.float64).reshape(-1, nI) if nI else None
    n_inst = L["n_instances"]
    R = np.zeros((nT, K))
    consts = np.zeros(nS + nI)
    consts[:nS] = sc

    def ld(i):
        if i < nT:
            return R[i]
        return np.full(K, consts[i - nT])

    def bits(v):
        return np.ascontiguousarray(v).view(np.int64)

    def run(ops, lo, hi):
        for (op, d, a, b, c) in ops[lo:hi]:
            va = ld(a)
            vb = ld(b)
            with np.errstate(all="ignore"):
                if op == "MOV": r = va.copy()
                elif op == "NEG": r = -va
                elif op == "NOT": r = np.where(va == 0.0, 1.0, 0.0)
                elif op == "ADD": r = va + vb
                elif op == "SUB": r = va - vb
                elif op == "MUL": r = va * vb
                elif op == "DIV": r = va / vb
                elif op == "LT": r = (va < vb).astype(np.float64)
                elif op == "LEQ": r = (va <= vb).astype(np.float64)
                elif op == "EQ": r = (va == vb).astype(np.float64)
                elif op == "AND": r = ((va != 0) & (vb != 0)).astype(np.float64)
                elif op == "OR": r = ((va != 0) | (vb != 0)).astype(np.float64)
                elif op == "SEL": r = np.where(va != 0.0, vb, ld(c))
                elif op == "IADD": r = (bits(va) + bits(vb)).view(np.float64)
                elif op == "ISUB": r = (bits(va) - bits(vb)).view(np.float64)
                elif op == "ILT": r = (bits(va) < bits(vb)).astype(np.float64)
                elif op == "ILEQ": r = (bits(va) <= bits(vb)).astype(np.float64)
                elif op == "IEQ": r = (bits(va) == bits(vb)).astype(np.float64)
                elif op == "MIN": r = np.fmin(va, vb)
                elif op == "MAX": r = np.fmax(va, vb)
                elif op == "MINP": r = np.minimum(va, vb)
                elif op == "MAXP": r = np.maximum(va, vb)
                elif op == "EFIRST": r = np.where(bits(va) != 0, va, vb)
                elif op == "EDIVZ":
                    r = np.where(va == 0.0, np.int64(c), np.int64(0)).astype(np.int64).view(np.float64)
                else:
                    raise ValueError(op)
            R[d] = r

    ops = L["ops"]
    for s, st in enumerate(L["steps"]):
        if st["begin"] < st["end"]:
            for j in range(nA):
                R[j] = S[:, s, j]
            run(ops, st["begin"], st["end"])
    lo, hi = L["inst_code"]
    n_days = len(L["outputs"])
    vals = np.zeros((K, n_inst * n_days))
    errs = np.zeros((K, n_inst * n_days), dtype=np.int64)
    for i in range(n_inst):
        if nI:
            consts[nS:] = inst[i]
        run(ops, lo, hi)
        for d, (v, e) in enumerate(L["outputs"]):
            vals[:, i * n_days + d] = ld(v)
            if e >= 0:
                errs[:, i * n_days + d] = bits(ld(e))
    return vals, errs


def spots_from_ext(L: dict, kernel: dict, model_order: list[str], ext: np.ndarray) -> np.ndarray:
    """Rebuild S[K][step][asset] from the reference's ext[K][row][col]."""
    days = L["days"]
    K = ext.shape[0]
    S = np.full((K, max(1, len(days)), L["n_assets"]), NAN)
    for r, day in enumerate(kernel["rows"]):
        s = days.index(day)
        for c, lab in enumerate(kernel["cols"]):
            S[:, s, model_order.index(lab)] = ext[:, r, c]
    return S
