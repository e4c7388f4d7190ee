"""ctypes binding of the engine's C ABI (include/cltk_b200.h).

Loads the in-tree ``libcltk_b200.so`` (built by ``make lib`` /
``__graft_entry__.build()``).  There is no fallback: if the library is
missing, importing the pricing API raises.
"""
from __future__ import annotations

import ctypes as C
import os

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("CLTK_B200_LIB") or os.path.join(HERE, "libcltk_b200.so")

# Every symbol include/cltk_b200.h declares (tests check the exports).
EXPORTS = [
    "cltk_version", "cltk_gpu_price", "cltk_gpu_price_batch", "cltk_plan_create",
    "cltk_plan_destroy", "cltk_plan_get_info", "cltk_plan_chunking", "cltk_plan_launch",
    "cltk_plan_finalize", "cltk_plan_error_word", "cltk_plan_set_error_word",
    "cltk_compile_listing", "cltk_plan_dump", "cltk_free", "cltk_debug_paths", "cltk_debug_rng", "cltk_debug_math",
    "cltk_fp64_peak", "cltk_black_scholes_call", "cltk_gpu_price_template",
    "cltk_kernel_literals", "cltk_plan_create_template", "cltk_gpu_price_ex",
    "cltk_plan_create_ex", "cltk_jit_source", "cltk_jit_compile", "cltk_reindex",
    "cltk_plan_create_batch_ex", "cltk_gpu_price_batch_ex", "cltk_plan_set_fault",
    "cltk_nccl_version", "cltk_debug_sobol",
]


MAX_DEVICES = 16  # CLTK_MAX_DEVICES


class OptionsC(C.Structure):
    _fields_ = [("device", C.c_int), ("rewrite", C.c_int), ("rng", C.c_int), ("jit", C.c_int),
                ("n_devices", C.c_int), ("devices", C.c_int * MAX_DEVICES),
                ("fault_inject", C.c_int), ("reserved", C.c_int * 3)]


class PriceResultC(C.Structure):
    _fields_ = [("price", C.c_double), ("std_error", C.c_double), ("paths", C.c_uint64),
                ("seed", C.c_uint64), ("valuation_day", C.c_uint64)]


class ErrorC(C.Structure):
    _fields_ = [("code", C.c_int), ("message", C.c_char * 504)]


class PlanInfoC(C.Structure):
    _fields_ = [(n, C.c_uint32) for n in (
        "n_assets", "n_steps", "n_thread", "n_shared_const", "n_inst_const", "n_instances",
        "n_days", "n_outputs", "n_shared_ops", "n_inst_ops", "has_err", "block")] + [
        ("kernel_nodes", C.c_uint64), ("dag_nodes", C.c_uint64), ("jit", C.c_uint32)]


_lib = None


def lib() -> C.CDLL:
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        raise ImportError(
            f"{LIB_PATH} is missing: build it with `make lib` or __graft_entry__.build(); "
            "the engine has no CPU fallback")
    L = C.CDLL(LIB_PATH)
    u64, u32, dbl, i32, vp, cp = C.c_uint64, C.c_uint32, C.c_double, C.c_int, C.c_void_p, C.c_char_p
    P64 = C.POINTER(u64)
    PD = C.POINTER(dbl)
    PR = C.POINTER(PriceResultC)
    PE = C.POINTER(ErrorC)
    L.cltk_version.restype = cp
    L.cltk_gpu_price.restype = i32
    L.cltk_gpu_price.argtypes = [cp, cp, u64, u64, P64, C.c_size_t, cp, C.c_uint, i32, PR, PE]
    L.cltk_gpu_price_batch.restype = i32
    L.cltk_gpu_price_batch.argtypes = [C.POINTER(cp), C.c_size_t, cp, u64, u64, P64, C.c_size_t,
                                       cp, i32, PR, PE]
    L.cltk_gpu_price_template.restype = i32
    L.cltk_gpu_price_template.argtypes = [cp, vp, C.c_size_t, C.c_size_t, cp, u64, u64, P64,
                                          C.c_size_t, cp, i32, PR, PE]
    L.cltk_kernel_literals.restype = i32
    L.cltk_kernel_literals.argtypes = [cp, vp, C.c_size_t, C.POINTER(C.c_size_t), PE]
    L.cltk_plan_create_template.restype = i32
    L.cltk_plan_create_template.argtypes = [cp, vp, C.c_size_t, C.c_size_t, cp, P64, C.c_size_t,
                                            cp, i32, i32, C.POINTER(vp), PE]
    L.cltk_plan_create.restype = i32
    L.cltk_plan_create.argtypes = [C.POINTER(cp), C.c_size_t, cp, P64, C.c_size_t, cp, i32, i32,
                                   C.POINTER(vp), PE]
    L.cltk_plan_destroy.argtypes = [vp]
    L.cltk_plan_get_info.restype = i32
    L.cltk_plan_get_info.argtypes = [vp, C.POINTER(PlanInfoC)]
    L.cltk_plan_chunking.restype = i32
    L.cltk_plan_chunking.argtypes = [vp, u64, P64, P64]
    L.cltk_plan_launch.restype = i32
    L.cltk_plan_launch.argtypes = [vp, u64, u64, u64, u64, vp, vp, PE]
    L.cltk_plan_finalize.restype = i32
    L.cltk_plan_finalize.argtypes = [vp, u64, u64, vp, P64, C.c_size_t, vp, PR, PE]
    L.cltk_plan_error_word.restype = i32
    L.cltk_plan_error_word.argtypes = [vp, vp, P64]
    L.cltk_plan_set_error_word.restype = i32
    L.cltk_plan_set_error_word.argtypes = [vp, vp, u64]
    L.cltk_compile_listing.restype = i32
    L.cltk_compile_listing.argtypes = [C.POINTER(cp), C.c_size_t, cp, P64, C.c_size_t, cp, i32,
                                       i32, C.POINTER(vp), PE]
    PO = C.POINTER(OptionsC)
    L.cltk_gpu_price_ex.restype = i32
    L.cltk_gpu_price_ex.argtypes = [cp, vp, C.c_size_t, C.c_size_t, cp, u64, u64, P64, C.c_size_t,
                                    cp, PO, PR, PE]
    L.cltk_plan_create_ex.restype = i32
    L.cltk_plan_create_ex.argtypes = [cp, vp, C.c_size_t, C.c_size_t, cp, P64, C.c_size_t, cp, PO,
                                      C.POINTER(vp), PE]
    L.cltk_reindex.restype = i32
    L.cltk_reindex.argtypes = [cp, cp, C.POINTER(vp), PE]
    L.cltk_jit_source.restype = i32
    L.cltk_jit_source.argtypes = [cp, vp, C.c_size_t, C.c_size_t, cp, P64, C.c_size_t, cp, i32, i32,
                                  C.POINTER(vp), PE]
    L.cltk_jit_compile.restype = i32
    L.cltk_jit_compile.argtypes = [cp, P64, C.POINTER(vp), PE]
    L.cltk_plan_create_batch_ex.restype = i32
    L.cltk_plan_create_batch_ex.argtypes = [C.POINTER(cp), C.c_size_t, cp, P64, C.c_size_t, cp, PO,
                                            C.POINTER(vp), PE]
    L.cltk_gpu_price_batch_ex.restype = i32
    L.cltk_gpu_price_batch_ex.argtypes = [C.POINTER(cp), C.c_size_t, cp, u64, u64, P64,
                                          C.c_size_t, cp, PO, PR, PE]
    L.cltk_plan_dump.restype = i32
    L.cltk_plan_dump.argtypes = [vp, C.POINTER(vp)]
    L.cltk_free.argtypes = [vp]
    L.cltk_debug_paths.restype = i32
    L.cltk_debug_paths.argtypes = [vp, u64, u64, u64, vp, vp, vp, P64, PE]
    L.cltk_debug_rng.restype = i32
    L.cltk_debug_rng.argtypes = [i32, u64, u64, u64, u64, vp, vp, vp, PE]
    L.cltk_debug_math.restype = i32
    L.cltk_debug_math.argtypes = [i32, i32, vp, u64, vp, PE]
    L.cltk_plan_set_fault.restype = i32
    L.cltk_plan_set_fault.argtypes = [vp, u64, u32, PE]
    L.cltk_nccl_version.restype = i32
    L.cltk_nccl_version.argtypes = [C.POINTER(i32), PE]
    L.cltk_debug_sobol.restype = i32
    L.cltk_debug_sobol.argtypes = [i32, u64, u64, u32, u32, i32, vp, PE]
    L.cltk_fp64_peak.restype = i32
    L.cltk_fp64_peak.argtypes = [i32, i32, PD, PD, PE]
    L.cltk_black_scholes_call.restype = dbl
    L.cltk_black_scholes_call.argtypes = [dbl] * 5
    _lib = L
    return L
