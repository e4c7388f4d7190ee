"""TEST INFRASTRUCTURE ONLY -- ctypes front for the two checkers.

* ``Ref``    -- the UNMODIFIED reference library compiled from
  /root/reference by oracle/Makefile (oracle/_ref/libcltkref.so, a prebuilt
  file on the GPU box).
* ``Oracle`` -- the repo's own C restatement (oracle/cltk_oracle.c).

Only tests/, bench.py's cpu_baseline / ``--impl reference`` legs and
``__graft_entry__.smoke()`` import this module, and only to CHECK the
product; the product path (paper_2108_03076_b200) never imports it.
"""
from __future__ import annotations

import ctypes as C
import json
import math
import os
from typing import Sequence

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
REF_SO = os.path.join(HERE, "_ref", "libcltkref.so")
ORACLE_SO = os.path.join(HERE, "_build", "libcltk_oracle.so")

# ---------------------------------------------------------------------------
# kernel JSON -> flat node array (layout of oracle_node in cltk_oracle.h)
# ---------------------------------------------------------------------------
NODE_DTYPE = np.dtype(
    [
        ("kind", "<i4"), ("op", "<i4"), ("a", "<i4"), ("b", "<i4"), ("c", "<i4"),
        ("pay_sign", "<i4"), ("row", "<u8"), ("col", "<u8"), ("nat", "<u8"),
        ("real", "<f8"), ("boolean", "<i4"), ("pad", "<i4"),
    ],
    align=True,
)
KINDS = {"if": 0, "float": 1, "nat": 2, "bool": 3, "now": 4, "timeref": 5,
         "obsref": 6, "payref": 7, "unop": 8, "binop": 9, "loopif": 10}
BINOPS = {"add": 0, "sub": 1, "mult": 2, "div": 3, "lt": 4, "leq": 5, "eq": 6,
          "and": 7, "or": 8}


def parties_of(kernel: dict) -> tuple[str, str]:
    """p1/p2 as priceAcrossTime picks them (proj/src/pricing.cpp:342-343)."""
    ps = kernel.get("parties", [])
    return (ps[0] if len(ps) > 0 else "you", ps[1] if len(ps) > 1 else "me")


def flatten_kernel(kernel: dict) -> tuple[np.ndarray, int]:
    p1, p2 = parties_of(kernel)
    nodes: list[tuple] = []

    def visit(e: dict) -> int:
        k = e["kind"]
        rec = dict(kind=KINDS[k], op=0, a=-1, b=-1, c=-1, pay_sign=0, row=0, col=0,
                   nat=0, real=0.0, boolean=0, pad=0)
        if k in ("if", "loopif"):
            rec["a"] = visit(e["cond"])
            rec["b"] = visit(e["then"])
            rec["c"] = visit(e["else"])
            if k == "loopif":
                rec["nat"] = int(e["window"])
        elif k == "float":
            rec["real"] = float(e["value"])
        elif k == "nat":
            rec["nat"] = int(e["value"])
        elif k == "bool":
            rec["boolean"] = int(bool(e["value"]))
        elif k == "timeref":
            rec["row"] = int(e["row"])
        elif k == "obsref":
            rec["row"] = int(e["row"])
            rec["col"] = int(e["col"])
        elif k == "payref":
            rec["row"] = int(e["row"])
            f, t = e["from"], e["to"]
            rec["pay_sign"] = 1 if (f == p1 and t == p2) else (-1 if (f == p2 and t == p1) else 0)
        elif k == "unop":
            rec["op"] = 0 if e["op"] == "neg" else 1
            rec["a"] = visit(e["arg"])
        elif k == "binop":
            rec["op"] = BINOPS[e["op"]]
            rec["a"] = visit(e["left"])
            rec["b"] = visit(e["right"])
        nodes.append(tuple(rec[n] for n in NODE_DTYPE.names))
        return len(nodes) - 1

    import sys
    old = sys.getrecursionlimit()
    sys.setrecursionlimit(max(old, 100000))
    try:
        root = visit(kernel["body"])
    finally:
        sys.setrecursionlimit(old)
    return np.array(nodes, dtype=NODE_DTYPE), root


class _OKernel(C.Structure):
    _fields_ = [("nodes", C.c_void_p), ("root", C.c_int32), ("n_rows", C.c_uint64),
                ("n_cols", C.c_uint64), ("rows", C.c_void_p)]


class _OModel(C.Structure):
    _fields_ = [("n_assets", C.c_uint64), ("spot", C.c_void_p), ("vol", C.c_void_p),
                ("drift", C.c_void_p), ("chol", C.c_void_p), ("rate", C.c_double),
                ("day_count", C.c_double), ("col_to_asset", C.c_void_p)]


class OracleError(RuntimeError):
    def __init__(self, code: int, msg: str):
        super().__init__(msg)
        self.code = code


def model_order(model: dict) -> list[str]:
    """modelFromJson's label order (proj/src/pricing.cpp:24-31)."""
    if "order" in model:
        return list(model["order"])
    return sorted(model["labels"].keys())


class Oracle:
    """The C restatement (oracle/cltk_oracle.c)."""

    def __init__(self, path: str = ORACLE_SO):
        if not os.path.exists(path):
            raise FileNotFoundError(f"{path} missing: run `make -C oracle oracle`")
        L = self.lib = C.CDLL(path)
        u64, dbl, i32 = C.c_uint64, C.c_double, C.c_int
        L.oracle_philox_bits.restype = u64
        L.oracle_philox_bits.argtypes = [u64, u64, u64]
        L.oracle_uniform.restype = dbl
        L.oracle_uniform.argtypes = [u64, u64, u64]
        L.oracle_inv_normal_cdf.restype = i32
        L.oracle_inv_normal_cdf.argtypes = [dbl, C.POINTER(dbl)]
        L.oracle_normal_cdf.restype = dbl
        L.oracle_normal_cdf.argtypes = [dbl]
        L.oracle_cholesky.restype = i32
        L.oracle_cholesky.argtypes = [C.c_void_p, i32, C.c_void_p]
        L.oracle_eval_kernel.restype = i32
        L.oracle_eval_kernel.argtypes = [C.POINTER(_OKernel), C.c_void_p, C.c_void_p, u64,
                                         C.POINTER(dbl), C.c_char_p, C.c_size_t]
        L.oracle_simulate_path.restype = i32
        L.oracle_simulate_path.argtypes = [C.POINTER(_OKernel), C.POINTER(_OModel), u64, u64,
                                           C.c_void_p]
        L.oracle_price.restype = i32
        L.oracle_price.argtypes = [C.POINTER(_OKernel), C.POINTER(_OModel), u64, u64, u64,
                                   C.c_void_p, u64, C.c_uint, C.c_void_p, C.c_void_p,
                                   C.c_void_p, C.c_char_p, C.c_size_t]

    # -- scalar functions ------------------------------------------------------
    def philox_bits(self, seed, path, i):
        return self.lib.oracle_philox_bits(seed, path, i)

    def uniform(self, seed, path, i):
        return self.lib.oracle_uniform(seed, path, i)

    def inv_normal_cdf(self, p):
        out = C.c_double()
        rc = self.lib.oracle_inv_normal_cdf(p, C.byref(out))
        if rc:
            raise OracleError(rc, "invNormalCdf domain error")
        return out.value

    def normal(self, seed, path, i):
        return self.inv_normal_cdf(self.uniform(seed, path, i))

    def normal_cdf(self, x):
        return self.lib.oracle_normal_cdf(x)

    def cholesky(self, m):
        a = np.ascontiguousarray(m, dtype=np.float64)
        n = a.shape[0]
        out = np.zeros_like(a)
        rc = self.lib.oracle_cholesky(a.ctypes.data, n, out.ctypes.data)
        if rc:
            raise OracleError(rc, "correlation matrix is not symmetric positive definite")
        return out

    # -- kernel / model marshalling --------------------------------------------
    def _kernel(self, kernel: dict):
        nodes, root = flatten_kernel(kernel)
        rows = np.ascontiguousarray(kernel["rows"], dtype=np.int64)
        ok = _OKernel(nodes.ctypes.data, root, len(kernel["rows"]), len(kernel["cols"]),
                      rows.ctypes.data)
        return ok, (nodes, rows)

    def _model(self, kernel: dict, model: dict):
        order = model_order(model)
        rate = float(model.get("rate", 0.0))
        labels = model["labels"]
        spot = np.array([float(labels[l]["spot"]) for l in order])
        vol = np.array([float(labels[l]["vol"]) for l in order])
        drift = np.array([float(labels[l].get("drift", rate)) for l in order])
        n = len(order)
        corr = model.get("corr", [])
        if not corr:
            chol = np.eye(n)
        else:
            if len(corr) != n:
                raise OracleError(5, "correlation matrix size does not match asset count")
            chol = self.cholesky(np.array(corr, dtype=np.float64))
        col_to_asset = []
        for lab in kernel["cols"]:
            if lab not in order:
                raise OracleError(5, "model has no asset spec for label " + lab)
            col_to_asset.append(order.index(lab))
        cta = np.array(col_to_asset + [0], dtype=np.uint64)
        chol = np.ascontiguousarray(chol)
        om = _OModel(n, spot.ctypes.data, vol.ctypes.data, drift.ctypes.data, chol.ctypes.data,
                     rate, float(model.get("dayCount", 365.0)), cta.ctypes.data)
        return om, (spot, vol, drift, chol, cta)

    def eval_kernel(self, kernel: dict, ext, disc, t_now: int) -> float:
        ok, keep = self._kernel(kernel)
        ext = np.ascontiguousarray(ext, dtype=np.float64)
        disc = np.ascontiguousarray(disc, dtype=np.float64)
        out = C.c_double()
        msg = C.create_string_buffer(256)
        rc = self.lib.oracle_eval_kernel(C.byref(ok), ext.ctypes.data, disc.ctypes.data,
                                         t_now, C.byref(out), msg, 256)
        if rc:
            raise OracleError(rc, msg.value.decode())
        return out.value

    def simulate_path(self, kernel: dict, model: dict, seed: int, path: int) -> np.ndarray:
        ok, k1 = self._kernel(kernel)
        om, k2 = self._model(kernel, model)
        ext = np.zeros((len(kernel["rows"]), len(kernel["cols"])))
        rc = self.lib.oracle_simulate_path(C.byref(ok), C.byref(om), seed, path, ext.ctypes.data)
        if rc:
            raise OracleError(rc, "oracle simulate_path failed")
        return ext

    def price(self, kernel: dict, model: dict, paths: int, seed: int,
              days: Sequence[int] = (0,), threads: int = 1, path0: int = 0,
              want_payoffs: bool = False):
        ok, k1 = self._kernel(kernel)
        om, k2 = self._model(kernel, model)
        d = np.ascontiguousarray(days, dtype=np.uint64)
        price = np.zeros(len(d))
        se = np.zeros(len(d))
        pay = np.zeros((len(d), paths)) if want_payoffs else None
        msg = C.create_string_buffer(256)
        rc = self.lib.oracle_price(C.byref(ok), C.byref(om), path0, paths, seed,
                                   d.ctypes.data, len(d), threads, price.ctypes.data,
                                   se.ctypes.data, pay.ctypes.data if pay is not None else None,
                                   msg, 256)
        if rc:
            raise OracleError(rc, msg.value.decode())
        out = [dict(price=float(price[i]), std_error=float(se[i]), paths=paths, seed=seed,
                    valuation_day=int(d[i])) for i in range(len(d))]
        return (out, pay) if want_payoffs else out


class Ref:
    """The compiled, unmodified reference (oracle/_ref/libcltkref.so)."""

    def __init__(self, path: str = REF_SO):
        if not os.path.exists(path):
            raise FileNotFoundError(f"{path} missing: run `make -C oracle ref` where "
                                    "/root/reference is mounted")
        L = self.lib = C.CDLL(path)
        u64, dbl, i32, vp = C.c_uint64, C.c_double, C.c_int, C.c_void_p
        L.cltkref_last_error.restype = C.c_char_p
        L.cltkref_free.argtypes = [vp]
        L.cltkref_compile_kernel_json.restype = i32
        L.cltkref_compile_kernel_json.argtypes = [C.c_char_p, C.c_char_p, i32, C.POINTER(vp)]
        L.cltkref_compile_il_json.restype = i32
        L.cltkref_compile_il_json.argtypes = [C.c_char_p, i32, C.POINTER(vp)]
        L.cltkref_reindex_json.restype = i32
        L.cltkref_reindex_json.argtypes = [C.c_char_p, C.c_char_p, C.POINTER(vp)]
        L.cltkref_kernel_source.restype = i32
        L.cltkref_kernel_source.argtypes = [C.c_char_p, C.POINTER(vp)]
        L.cltkref_philox_bits.restype = u64
        L.cltkref_philox_bits.argtypes = [u64, u64, u64]
        L.cltkref_uniform.restype = dbl
        L.cltkref_uniform.argtypes = [u64, u64, u64]
        L.cltkref_normal.restype = i32
        L.cltkref_normal.argtypes = [u64, u64, u64, C.POINTER(dbl)]
        L.cltkref_inv_normal_cdf.restype = i32
        L.cltkref_inv_normal_cdf.argtypes = [dbl, C.POINTER(dbl)]
        L.cltkref_normal_cdf.restype = dbl
        L.cltkref_normal_cdf.argtypes = [dbl]
        L.cltkref_black_scholes_call.restype = dbl
        L.cltkref_black_scholes_call.argtypes = [dbl] * 5
        L.cltkref_cholesky.restype = i32
        L.cltkref_cholesky.argtypes = [vp, i32, vp]
        L.cltkref_kernel_load.restype = i32
        L.cltkref_kernel_load.argtypes = [C.c_char_p, C.POINTER(vp)]
        L.cltkref_kernel_free.argtypes = [vp]
        L.cltkref_kernel_shape.argtypes = [vp, C.POINTER(u64), C.POINTER(u64)]
        L.cltkref_model_load.restype = i32
        L.cltkref_model_load.argtypes = [C.c_char_p, C.POINTER(vp)]
        L.cltkref_model_free.argtypes = [vp]
        L.cltkref_simulate_paths.restype = i32
        L.cltkref_simulate_paths.argtypes = [vp, vp, u64, u64, u64, vp]
        L.cltkref_disc.restype = i32
        L.cltkref_disc.argtypes = [vp, vp, vp]
        L.cltkref_eval_kernel.restype = i32
        L.cltkref_eval_kernel.argtypes = [vp, vp, vp, u64, C.c_char_p, C.c_char_p,
                                          C.POINTER(dbl)]
        L.cltkref_path_payoffs.restype = i32
        L.cltkref_path_payoffs.argtypes = [vp, vp, u64, u64, u64, vp, u64, vp]
        L.cltkref_price.restype = i32
        L.cltkref_price.argtypes = [vp, vp, u64, u64, vp, u64, C.c_char_p, C.c_uint, vp, vp]

    def _check(self, rc):
        if rc:
            raise OracleError(rc, self.lib.cltkref_last_error().decode())

    def _take_string(self, p) -> str:
        s = C.cast(p, C.c_char_p).value.decode()
        self.lib.cltkref_free(p)
        return s

    def compile_kernel(self, contract_src: str, tenv: dict | None = None, cut: bool = True) -> dict:
        out = C.c_void_p()
        self._check(self.lib.cltkref_compile_kernel_json(
            contract_src.encode(), json.dumps(tenv or {}).encode(), int(cut), C.byref(out)))
        return json.loads(self._take_string(out))

    def compile_il(self, contract_src: str, cut: bool = True) -> dict:
        """ilToJson(cutPayoff?(compileContract(parse(src)))) -- reindex's input."""
        out = C.c_void_p()
        self._check(self.lib.cltkref_compile_il_json(contract_src.encode(), int(cut), C.byref(out)))
        return json.loads(self._take_string(out))

    def reindex(self, il: dict, tenv: dict | None = None) -> dict:
        out = C.c_void_p()
        self._check(self.lib.cltkref_reindex_json(json.dumps(il).encode(),
                                                  json.dumps(tenv or {}).encode(), C.byref(out)))
        return json.loads(self._take_string(out))

    def kernel_source(self, kernel: dict) -> str:
        out = C.c_void_p()
        self._check(self.lib.cltkref_kernel_source(json.dumps(kernel).encode(), C.byref(out)))
        return self._take_string(out)

    def philox_bits(self, seed, path, i):
        return self.lib.cltkref_philox_bits(seed, path, i)

    def uniform(self, seed, path, i):
        return self.lib.cltkref_uniform(seed, path, i)

    def normal(self, seed, path, i):
        out = C.c_double()
        self._check(self.lib.cltkref_normal(seed, path, i, C.byref(out)))
        return out.value

    def inv_normal_cdf(self, p):
        out = C.c_double()
        self._check(self.lib.cltkref_inv_normal_cdf(p, C.byref(out)))
        return out.value

    def normal_cdf(self, x):
        return self.lib.cltkref_normal_cdf(x)

    def black_scholes_call(self, spot, strike, rate, vol, t):
        return self.lib.cltkref_black_scholes_call(spot, strike, rate, vol, t)

    def cholesky(self, m):
        a = np.ascontiguousarray(m, dtype=np.float64)
        out = np.zeros_like(a)
        self._check(self.lib.cltkref_cholesky(a.ctypes.data, a.shape[0], out.ctypes.data))
        return out

    class _Handles:
        def __init__(self, ref, kernel, model):
            self.ref = ref
            self.k = C.c_void_p()
            self.m = C.c_void_p()
            ref._check(ref.lib.cltkref_kernel_load(json.dumps(kernel).encode(), C.byref(self.k)))
            if model is not None:
                ref._check(ref.lib.cltkref_model_load(json.dumps(model).encode(), C.byref(self.m)))

        def __enter__(self):
            return self

        def __exit__(self, *a):
            self.ref.lib.cltkref_kernel_free(self.k)
            if self.m:
                self.ref.lib.cltkref_model_free(self.m)

    def simulate_paths(self, kernel, model, seed, path0, npaths) -> np.ndarray:
        R, Cc = len(kernel["rows"]), len(kernel["cols"])
        out = np.zeros((npaths, R, Cc))
        with self._Handles(self, kernel, model) as h:
            self._check(self.lib.cltkref_simulate_paths(h.k, h.m, seed, path0, npaths,
                                                        out.ctypes.data))
        return out

    def disc(self, kernel, model) -> np.ndarray:
        out = np.zeros(len(kernel["rows"]))
        with self._Handles(self, kernel, model) as h:
            self._check(self.lib.cltkref_disc(h.k, h.m, out.ctypes.data))
        return out

    def eval_kernel(self, kernel, ext, disc, t_now, p1=None, p2=None) -> float:
        q1, q2 = parties_of(kernel)
        ext = np.ascontiguousarray(ext, dtype=np.float64)
        disc = np.ascontiguousarray(disc, dtype=np.float64)
        out = C.c_double()
        with self._Handles(self, kernel, None) as h:
            self._check(self.lib.cltkref_eval_kernel(h.k, ext.ctypes.data, disc.ctypes.data,
                                                     t_now, (p1 or q1).encode(),
                                                     (p2 or q2).encode(), C.byref(out)))
        return out.value

    def path_payoffs(self, kernel, model, seed, path0, npaths, days=(0,)) -> np.ndarray:
        d = np.ascontiguousarray(days, dtype=np.uint64)
        out = np.zeros((npaths, len(d)))
        with self._Handles(self, kernel, model) as h:
            self._check(self.lib.cltkref_path_payoffs(h.k, h.m, seed, path0, npaths,
                                                      d.ctypes.data, len(d), out.ctypes.data))
        return out

    def price(self, kernel, model, paths, seed, days=(0,), tenv=None, threads=0):
        d = np.ascontiguousarray(days, dtype=np.uint64)
        pr = np.zeros(len(d))
        se = np.zeros(len(d))
        with self._Handles(self, kernel, model) as h:
            self._check(self.lib.cltkref_price(h.k, h.m, paths, seed, d.ctypes.data, len(d),
                                               json.dumps(tenv or {}).encode(), threads,
                                               pr.ctypes.data, se.ctypes.data))
        return [dict(price=float(pr[i]), std_error=float(se[i]), paths=paths, seed=seed,
                     valuation_day=int(d[i])) for i in range(len(d))]


def ref_available() -> bool:
    return os.path.exists(REF_SO)


def black_scholes_call(spot, strike, rate, vol, t):
    """Closed form, proj/src/pricing.cpp:150-159 (math.erfc is glibc's)."""
    if t <= 0.0:
        return max(spot - strike, 0.0)
    ncdf = lambda x: 0.5 * math.erfc(-x / math.sqrt(2.0))
    sd = vol * math.sqrt(t)
    d1 = (math.log(spot / strike) + (rate + 0.5 * vol * vol) * t) / sd
    d2 = d1 - sd
    return spot * ncdf(d1) - strike * math.exp(-rate * t) * ncdf(d2)
