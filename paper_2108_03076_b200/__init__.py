"""B200-native Monte Carlo pricing of compiled contract kernels.

The Python face of the engine mirrors the reference's pybind module
(``cltk``, proj/python/bindings.cpp) for the pricing path:

================================  ==============================================
reference (``cltk``)              here
================================  ==============================================
``price(kernel, model, paths=100000, seed=0, days=[0], tenv={}, threads=0)``
                                  same signature and result dicts
                                  (bindings.cpp:103-126)
``black_scholes_call``            same (bindings.cpp:128-129)
``Kernel.rows`` / ``.cols``       same (bindings.cpp:75-80)
``ContractError`` /               same hierarchy (bindings.cpp:47-49); eval
``ContractParseError`` /          errors raise ``ContractError`` with
``ContractTypeError``             ``.code == 5``, as the reference's do
================================  ==============================================

Kernels are the reference's flattened payoffs in its own wire format
(``kernelToJson``, proj/src/kernel.cpp:620); the contract front end
(parse/compile/cutPayoff/reindex) stays the reference's.  Everything below
runs through ``libcltk_b200.so`` (sm_100a kernels + C++ host); there is no
CPU fallback.
"""
from __future__ import annotations

import ctypes as C
import json
import os
import sys
from typing import Any, Iterable, Sequence

from . import _native

__all__ = [
    "Kernel", "ContractError", "ContractParseError", "ContractTypeError",
    "ContractUnsupportedError", "price", "price_batch", "black_scholes_call", "Plan",
    "compile_listing", "debug_rng", "debug_math", "fp64_peak", "load_kernel", "version",
    "kernel_literals", "price_template", "jit_source", "jit_compile", "reindex",
    "debug_sobol", "nccl_version",
]


class ContractError(Exception):
    """cltk::Error (proj/include/cltk/errors.hpp:20-30); ``code`` = ErrorCode."""

    def __init__(self, message: str, code: int = 5):
        super().__init__(message)
        self.code = code


class ContractParseError(ContractError):
    pass


class ContractTypeError(ContractError):
    pass


class ContractUnsupportedError(ContractError):
    pass


def _raise(code: int, err: _native.ErrorC) -> None:
    if code == 0:
        return
    msg = err.message.decode(errors="replace")
    cls = {2: ContractParseError, 3: ContractTypeError, 4: ContractUnsupportedError}.get(
        code, ContractError)
    raise cls(msg, code)


def _deep(fn, *a):
    old = sys.getrecursionlimit()
    sys.setrecursionlimit(max(old, 200000))
    try:
        return fn(*a)
    finally:
        sys.setrecursionlimit(old)


class Kernel:
    """A flattened payoff kernel (cltk::Kernel, proj/include/cltk/kernel.hpp:71-79)
    held in the reference's JSON wire format."""

    def __init__(self, source: str | dict):
        """``source``: the kernel JSON (kernelToJson, dict or text) or the
        reference's textual kernel format (emitKernelSource)."""
        if isinstance(source, dict):
            self._obj = source
            self._json = _deep(json.dumps, source)
        elif source.lstrip().startswith("{"):
            self._json = source
            self._obj = _deep(json.loads, source)
        else:  # kernel text: the engine reads it natively; header parsed here
            import re
            self._json = source
            rows = re.search(r"let rows = \[([^\]]*)\]", source)
            cols = re.search(r"let cols = \[([^\]]*)\]", source)
            if not rows or not cols:
                raise ContractParseError("kernel source: missing rows/cols header", 2)
            r = [int(x) for x in rows.group(1).split(",") if x.strip()]
            self._obj = {"rows": r, "cols": re.findall(r'"([^"]*)"', cols.group(1)),
                         "tvars": [], "parties": list(dict.fromkeys(
                             re.findall(r"pay\[[^,]+, *(\w+), *(\w+)\]", source) and
                             [p for pr in re.findall(r"pay\[[^,]+, *(\w+), *(\w+)\]", source)
                              for p in pr])),
                         "horizon": (max(r) + 1) if r else 1, "body": None}

    @classmethod
    def from_file(cls, path: str) -> "Kernel":
        with open(path) as f:
            return cls(f.read())

    @property
    def json(self) -> str:
        return self._json

    @property
    def obj(self) -> dict:
        return self._obj

    rows = property(lambda self: list(self._obj["rows"]))
    cols = property(lambda self: list(self._obj["cols"]))
    tvars = property(lambda self: list(self._obj["tvars"]))
    parties = property(lambda self: list(self._obj["parties"]))
    horizon = property(lambda self: int(self._obj["horizon"]))

    def literals(self) -> list[float]:
        """FloatLit values in postorder (the order the engine's literal pool uses)."""
        if self._obj.get("body") is None:
            return kernel_literals(self._json)
        out: list[float] = []

        def walk(e):
            stack = [(e, False)]
            while stack:
                node, done = stack.pop()
                k = node["kind"]
                if done or k not in ("if", "loopif", "unop", "binop"):
                    if k == "float":
                        out.append(float(node["value"]))
                    continue
                stack.append((node, True))
                kids = ([node["cond"], node["then"], node["else"]] if k in ("if", "loopif")
                        else [node["arg"]] if k == "unop" else [node["left"], node["right"]])
                for c in reversed(kids):
                    stack.append((c, False))
        walk(self._obj["body"])
        return out

    def with_literals(self, mapping: dict[float, float]) -> "Kernel":
        """A new instance of the same template with FloatLit values substituted
        (``{old_value: new_value}``): the "templated contract batch" input."""

        def sub(e):
            stack = [e]
            while stack:
                node = stack.pop()
                k = node["kind"]
                if k == "float":
                    v = float(node["value"])
                    if v in mapping:
                        node["value"] = float(mapping[v])
                elif k in ("if", "loopif"):
                    stack += [node["cond"], node["then"], node["else"]]
                elif k == "unop":
                    stack.append(node["arg"])
                elif k == "binop":
                    stack += [node["left"], node["right"]]
        obj = _deep(json.loads, self._json)
        sub(obj["body"])
        return Kernel(obj)


def load_kernel(path: str) -> Kernel:
    return Kernel.from_file(path)


def _kernel_json(k: Kernel | str | dict) -> bytes:
    if isinstance(k, Kernel):
        return k.json.encode()
    if isinstance(k, dict):
        return _deep(json.dumps, k).encode()
    return k.encode()


def _model_json(m: str | dict) -> bytes:
    return (m if isinstance(m, str) else json.dumps(m)).encode()


def _tenv_json(t: dict | None) -> bytes:
    return json.dumps(t or {}).encode()


def _days(days: Iterable[int]):
    d = [int(x) for x in days]
    return (C.c_uint64 * max(1, len(d)))(*d), len(d)


def _results(arr, n: int) -> list[dict]:
    out = []
    for i in range(n):
        r = arr[i]  # (one struct view per result: field access is the slow part)
        out.append({"price": r.price, "std_error": r.std_error, "paths": r.paths,
                    "seed": r.seed, "valuation_day": r.valuation_day})
    return out


RNG_MODES = {"philox": 0, "sobol": 1}
# payoff evaluation: bytecode interpreter / NVRTC-generated kernel / NVRTC when
# available and the program is small (results are bit-identical)
JIT_MODES = {False: 0, True: 1, "auto": 2}


def _options(device: int = -1, rewrite: bool = True, rng: str = "philox", jit="auto",
             devices: Sequence[int] | None = None, fault: bool = False):
    if rng not in RNG_MODES:
        raise ValueError(f"rng must be one of {sorted(RNG_MODES)}")
    if jit not in JIT_MODES:
        raise ValueError("jit must be False, True or 'auto'")
    o = _native.OptionsC()
    o.device, o.rewrite, o.rng = int(device), int(bool(rewrite)), RNG_MODES[rng]
    o.jit = JIT_MODES[jit]
    devs = [int(d) for d in (devices or [])]
    if len(devs) > _native.MAX_DEVICES:
        raise ValueError(f"at most {_native.MAX_DEVICES} devices")
    o.n_devices = len(devs)
    for i, d in enumerate(devs):
        o.devices[i] = d
    o.fault_inject = int(bool(fault))
    return o


def version() -> str:
    return _native.lib().cltk_version().decode()


def price(kernel: Kernel | str | dict, model: str | dict, paths: int = 100000, seed: int = 0,
          days: Sequence[int] = (0,), tenv: dict | None = None, threads: int = 0,
          device: int = -1, rng: str = "philox", jit="auto",
          devices: Sequence[int] | None = None) -> list[dict]:
    """priceAcrossTime on the GPU (cltk.price, proj/python/bindings.cpp:103-126).

    Returns one dict per valuation day: ``price``, ``std_error``, ``paths``,
    ``seed``, ``valuation_day``.  ``threads`` is accepted for compatibility
    (results never depend on it).  ``rng="philox"`` (default) reproduces the
    reference's per-path values bit for bit; ``rng="sobol"`` is the QMC mode
    (Sobol + AS241 + Brownian bridge).  ``jit``: ``"auto"`` (default) evaluates
    the payoff with the NVRTC-generated kernel when NVRTC is available (compiled
    once per program shape and cached in-process and on disk), ``True`` always,
    ``False`` with the bytecode interpreter -- bit-identical results.
    ``devices``: shard the call over these GPUs of this process (one NCCL
    all-gather of the chunk partials; bit-identical to one GPU); default: the
    GPUs ``$CLTK_DEVICES`` lists, else ``device``."""
    L = _native.lib()
    d, nd = _days(days)
    out = (_native.PriceResultC * max(1, nd))()
    err = _native.ErrorC()
    if rng == "philox" and jit == "auto" and not devices:
        rc = L.cltk_gpu_price(_kernel_json(kernel), _model_json(model), int(paths), int(seed), d,
                              nd, _tenv_json(tenv), int(threads), int(device), out, C.byref(err))
    else:
        o = _options(device, True, rng, jit, devices)
        rc = L.cltk_gpu_price_ex(_kernel_json(kernel), None, 1, 0, _model_json(model), int(paths),
                                 int(seed), d, nd, _tenv_json(tenv), C.byref(o), out,
                                 C.byref(err))
    _raise(rc, err)
    return _results(out, nd)


def price_batch(kernels: Sequence[Kernel | str | dict], model: str | dict, paths: int = 100000,
                seed: int = 0, days: Sequence[int] = (0,), tenv: dict | None = None,
                device: int = -1, rng: str = "philox", jit="auto",
                devices: Sequence[int] | None = None) -> list[list[dict]]:
    """Price literal instances of one template on one shared path set (no
    recompilation per instance): ``[instance][day]`` result dicts."""
    L = _native.lib()
    d, nd = _days(days)
    n = len(kernels)
    arr = (C.c_char_p * n)(*[_kernel_json(k) for k in kernels])
    out = (_native.PriceResultC * max(1, n * nd))()
    err = _native.ErrorC()
    if rng == "philox" and jit == "auto" and not devices:
        rc = L.cltk_gpu_price_batch(arr, n, _model_json(model), int(paths), int(seed), d, nd,
                                    _tenv_json(tenv), int(device), out, C.byref(err))
    else:
        o = _options(device, True, rng, jit, devices)
        rc = L.cltk_gpu_price_batch_ex(arr, n, _model_json(model), int(paths), int(seed), d, nd,
                                       _tenv_json(tenv), C.byref(o), out, C.byref(err))
    _raise(rc, err)
    flat = _results(out, n * nd)
    return [flat[i * nd:(i + 1) * nd] for i in range(n)]


def kernel_literals(kernel: Kernel | str | dict) -> list[float]:
    """The kernel's float literals in the engine's template order (host only)."""
    import numpy as np
    L = _native.lib()
    kj = _kernel_json(kernel)
    n = C.c_size_t()
    err = _native.ErrorC()
    _raise(L.cltk_kernel_literals(kj, None, 0, C.byref(n), C.byref(err)), err)
    out = np.zeros(max(1, n.value))
    _raise(L.cltk_kernel_literals(kj, out.ctypes.data, n.value, C.byref(n), C.byref(err)), err)
    return [float(x) for x in out[:n.value]]


def price_template(kernel: Kernel | str | dict, literals, model: str | dict,
                   paths: int = 100000, seed: int = 0, days: Sequence[int] = (0,),
                   tenv: dict | None = None, device: int = -1,
                   rng: str = "philox", jit="auto",
                   devices: Sequence[int] | None = None) -> list[list[dict]]:
    """Price instances of one template given as a literal table
    ``literals[instance][j]`` (j in ``kernel_literals`` order): one compile,
    one path set, the literals passed to the kernel as data."""
    import numpy as np
    lit = np.ascontiguousarray(literals, dtype=np.float64)
    if lit.ndim != 2:
        raise ValueError("literals must be [n_instances][n_literals]")
    L = _native.lib()
    d, nd = _days(days)
    n = lit.shape[0]
    out = (_native.PriceResultC * max(1, n * nd))()
    err = _native.ErrorC()
    o = _options(device, True, rng, jit, devices)
    rc = L.cltk_gpu_price_ex(_kernel_json(kernel), lit.ctypes.data, n, lit.shape[1],
                             _model_json(model), int(paths), int(seed), d, nd, _tenv_json(tenv),
                             C.byref(o), out, C.byref(err))
    _raise(rc, err)
    flat = _results(out, n * nd)
    return [flat[i * nd:(i + 1) * nd] for i in range(n)]


def black_scholes_call(spot: float, strike: float, rate: float, vol: float,
                       expiry: float) -> float:
    return _native.lib().cltk_black_scholes_call(spot, strike, rate, vol, expiry)


def compile_listing(kernels: Sequence[Kernel | str | dict] | Kernel, model: str | dict,
                    days: Sequence[int] = (0,), tenv: dict | None = None,
                    rewrite: bool = True, rng: str = "philox") -> dict:
    """Host-only compile: the streaming device program as JSON (no GPU needed)."""
    if not isinstance(kernels, (list, tuple)):
        kernels = [kernels]
    L = _native.lib()
    d, nd = _days(days)
    arr = (C.c_char_p * len(kernels))(*[_kernel_json(k) for k in kernels])
    out = C.c_void_p()
    err = _native.ErrorC()
    rc = L.cltk_compile_listing(arr, len(kernels), _model_json(model), d, nd, _tenv_json(tenv),
                                int(rewrite), RNG_MODES[rng], C.byref(out), C.byref(err))
    _raise(rc, err)
    s = C.cast(out, C.c_char_p).value.decode()
    L.cltk_free(out)
    return _deep(json.loads, s)


def reindex(il: str | dict, tenv: dict | None = None) -> Kernel:
    """reindex (proj/src/kernel.cpp:301-303): the IL of a compiled contract
    (its JSON wire format, ``ilToJson``) flattened into a pricing kernel, the
    template variables bound from ``tenv``.  Host only."""
    L = _native.lib()
    ij = (il if isinstance(il, str) else json.dumps(il)).encode()
    out = C.c_void_p()
    err = _native.ErrorC()
    _raise(L.cltk_reindex(ij, _tenv_json(tenv), C.byref(out), C.byref(err)), err)
    s = C.cast(out, C.c_char_p).value.decode()
    L.cltk_free(out)
    return Kernel(s)


def jit_source(kernel: Kernel | str | dict, model: str | dict, days: Sequence[int] = (0,),
               tenv: dict | None = None, rewrite: bool = True, rng: str = "philox",
               literals=None) -> str:
    """Host-only: the CUDA source of the NVRTC payoff kernel for this program
    (``literals``: optional template literal table, as in ``price_template``)."""
    import numpy as np
    L = _native.lib()
    d, nd = _days(days)
    out = C.c_void_p()
    err = _native.ErrorC()
    if literals is not None:
        lit = np.ascontiguousarray(literals, dtype=np.float64)
        lp, n_i, n_l = lit.ctypes.data, lit.shape[0], lit.shape[1]
    else:
        lit, lp, n_i, n_l = None, None, 1, 0
    rc = L.cltk_jit_source(_kernel_json(kernel), lp, n_i, n_l, _model_json(model), d, nd,
                           _tenv_json(tenv), int(rewrite), RNG_MODES[rng], C.byref(out),
                           C.byref(err))
    _raise(rc, err)
    s = C.cast(out, C.c_char_p).value.decode()
    L.cltk_free(out)
    return s


def jit_compile(source: str) -> tuple[int, str]:
    """Host-only NVRTC compile of a generated source for sm_100a:
    (cubin bytes, compiler log).  Raises UnsupportedError on failure."""
    L = _native.lib()
    n = C.c_uint64()
    out = C.c_void_p()
    err = _native.ErrorC()
    rc = L.cltk_jit_compile(source.encode(), C.byref(n), C.byref(out), C.byref(err))
    _raise(rc, err)
    log = C.cast(out, C.c_char_p).value.decode()
    L.cltk_free(out)
    return n.value, log


class Plan:
    """Compiled plan on one device: the building block of multi-GPU pricing
    (see ``paper_2108_03076_b200.distributed``)."""

    def __init__(self, kernels: Sequence[Kernel | str | dict] | Kernel, model: str | dict,
                 days: Sequence[int] = (0,), tenv: dict | None = None, device: int = -1,
                 rewrite: bool = True, literals=None, rng: str = "philox", jit=False,
                 fault: bool = False):
        """``fault=True`` (tests): the kernel with the fault hook compiled in
        (``set_fault``)."""
        if not isinstance(kernels, (list, tuple)):
            kernels = [kernels]
        self._L = _native.lib()
        self.days = [int(x) for x in days]
        d, nd = _days(self.days)
        self._h = C.c_void_p()
        err = _native.ErrorC()
        if literals is not None:
            import numpy as np
            o = _options(device, rewrite, rng, jit, fault=fault)
            lit = np.ascontiguousarray(literals, dtype=np.float64)
            lp, n_i, n_l = lit.ctypes.data, lit.shape[0], lit.shape[1]
            if len(kernels) != 1:
                raise ValueError("literal-table plans take one template kernel")
            rc = self._L.cltk_plan_create_ex(
                _kernel_json(kernels[0]), lp, n_i, n_l, _model_json(model), d, nd,
                _tenv_json(tenv), C.byref(o), C.byref(self._h), C.byref(err))
        else:
            arr = (C.c_char_p * len(kernels))(*[_kernel_json(k) for k in kernels])
            o = _options(device, rewrite, rng, jit, fault=fault)
            rc = self._L.cltk_plan_create_batch_ex(arr, len(kernels), _model_json(model), d, nd,
                                                   _tenv_json(tenv), C.byref(o),
                                                   C.byref(self._h), C.byref(err))
        _raise(rc, err)
        info = _native.PlanInfoC()
        self._L.cltk_plan_get_info(self._h, C.byref(info))
        self.info = {n: getattr(info, n) for n, _ in _native.PlanInfoC._fields_}

    def close(self) -> None:
        if getattr(self, "_h", None):
            self._L.cltk_plan_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    @property
    def n_outputs(self) -> int:
        return int(self.info["n_outputs"])

    def chunking(self, paths: int) -> tuple[int, int]:
        cp, nc = C.c_uint64(), C.c_uint64()
        self._L.cltk_plan_chunking(self._h, int(paths), C.byref(cp), C.byref(nc))
        return cp.value, nc.value

    def launch(self, paths: int, seed: int, c0: int, c1: int, partials_ptr: int,
               stream_ptr: int = 0) -> None:
        err = _native.ErrorC()
        rc = self._L.cltk_plan_launch(self._h, int(paths), int(seed), int(c0), int(c1),
                                      C.c_void_p(partials_ptr), C.c_void_p(stream_ptr),
                                      C.byref(err))
        _raise(rc, err)

    def finalize(self, paths: int, seed: int, partials_ptr: int, stream_ptr: int = 0) -> list[dict]:
        d, nd = _days(self.days)
        n = self.n_outputs
        out = (_native.PriceResultC * max(1, n))()
        err = _native.ErrorC()
        rc = self._L.cltk_plan_finalize(self._h, int(paths), int(seed), C.c_void_p(partials_ptr),
                                        d, nd, C.c_void_p(stream_ptr), out, C.byref(err))
        _raise(rc, err)
        return _results(out, n)

    def set_fault(self, path: int, draw: int) -> None:
        """Test hook (plans built with ``fault=True``): later launches force
        the uniform of ``draw`` of ``path`` to exactly 1.0 -- the reference's
        invNormalCdf domain error.  ``path=-1``: none."""
        err = _native.ErrorC()
        rc = self._L.cltk_plan_set_fault(self._h, int(path) & (2**64 - 1), int(draw), C.byref(err))
        _raise(rc, err)

    def error_word(self, stream_ptr: int = 0) -> int:
        w = C.c_uint64()
        self._L.cltk_plan_error_word(self._h, C.c_void_p(stream_ptr), C.byref(w))
        return w.value

    def set_error_word(self, word: int, stream_ptr: int = 0) -> None:
        self._L.cltk_plan_set_error_word(self._h, C.c_void_p(stream_ptr), C.c_uint64(word))

    def dump(self) -> dict:
        out = C.c_void_p()
        self._L.cltk_plan_dump(self._h, C.byref(out))
        s = C.cast(out, C.c_char_p).value.decode()
        self._L.cltk_free(out)
        return json.loads(s)

    def debug_paths(self, seed: int, path0: int, npaths: int, spots: bool = False,
                    normals: bool = False):
        """Per-path outputs [npaths][n_outputs] (and optionally the simulated
        spots / normals [npaths][n_steps][n_assets]) from the same device code."""
        import numpy as np
        ns, na = int(self.info["n_steps"]), max(1, int(self.info["n_assets"]))
        outs = np.zeros((npaths, self.n_outputs))
        S = np.zeros((npaths, ns, na)) if spots else None
        Z = np.zeros((npaths, ns, na)) if normals else None
        w = C.c_uint64()
        err = _native.ErrorC()
        rc = self._L.cltk_debug_paths(self._h, int(seed), int(path0), int(npaths),
                                      outs.ctypes.data, S.ctypes.data if S is not None else None,
                                      Z.ctypes.data if Z is not None else None, C.byref(w),
                                      C.byref(err))
        _raise(rc, err)
        return outs, S, Z, w.value


def debug_rng(seed: int, path: int, i0: int, n: int, device: int = -1):
    """Philox bits / uniforms / normals of CounterRng(seed, path) indices
    [i0, i0+n), computed by the device code the pricing kernel uses."""
    import numpy as np
    bits = np.zeros(n, dtype=np.uint64)
    uni = np.zeros(n)
    nor = np.zeros(n)
    err = _native.ErrorC()
    rc = _native.lib().cltk_debug_rng(int(device), int(seed), int(path), int(i0), int(n),
                                      bits.ctypes.data, uni.ctypes.data, nor.ctypes.data,
                                      C.byref(err))
    _raise(rc, err)
    return bits, uni, nor


def debug_math(fn: str, x, device: int = -1):
    """Device build of the engine's glibc-exact ``exp`` / ``log`` / ``erfc`` or
    the reference's ``inv_normal`` (invNormalCdf) over an array; ``div``
    (pairs ``x[2i] / x[2i+1]`` through the engine's bounded-range division,
    written to both slots) and ``halley_arg`` (``-x / sqrt(2.0)``) check the
    engine's division shortcuts against IEEE; ``log_fmin`` / ``log_fmax``
    (pairs ``(m, x)``: ``exp`` of the running minimum / maximum the NVRTC
    payoff code keeps in the log domain, both slots) against
    ``fmin(exp(m), exp(x))`` / ``fmax``."""
    import numpy as np
    code = {"exp": 0, "log": 1, "erfc": 2, "inv_normal": 3, "div": 4, "halley_arg": 5,
            "log_fmin": 6, "log_fmax": 7, "log_fmin_b": 8, "log_fmax_b": 9}[fn]
    x = np.ascontiguousarray(x, dtype=np.float64)
    out = np.zeros_like(x)
    err = _native.ErrorC()
    rc = _native.lib().cltk_debug_math(int(device), code, x.ctypes.data, len(x), out.ctypes.data,
                                       C.byref(err))
    _raise(rc, err)
    return out


def debug_sobol(n0: int, n: int, d0: int, nd: int, aligned: bool = True, device: int = -1):
    """Sobol integers [n][nd] of points n0.. and dimensions d0.. from the
    device generator of the QMC mode (``aligned``: its warp-cooperative
    skip-ahead, n0 % 32 == 0)."""
    import numpy as np
    out = np.zeros((n, nd), dtype=np.uint32)
    err = _native.ErrorC()
    rc = _native.lib().cltk_debug_sobol(int(device), int(n0), int(n), int(d0), int(nd),
                                        int(bool(aligned)), out.ctypes.data, C.byref(err))
    _raise(rc, err)
    return out


def nccl_version() -> int:
    """NCCL version code the in-process multi-GPU path loads (raises
    ContractUnsupportedError when libnccl.so.2 is not loadable)."""
    v = C.c_int()
    err = _native.ErrorC()
    _raise(_native.lib().cltk_nccl_version(C.byref(v), C.byref(err)), err)
    return v.value


def fp64_peak(device: int = -1, iters: int = 4096) -> tuple[float, float]:
    """Measured DFMA throughput in TFLOP/s (and the seconds it took)."""
    t, s = C.c_double(), C.c_double()
    err = _native.ErrorC()
    rc = _native.lib().cltk_fp64_peak(int(device), int(iters), C.byref(t), C.byref(s),
                                      C.byref(err))
    _raise(rc, err)
    return t.value, s.value
