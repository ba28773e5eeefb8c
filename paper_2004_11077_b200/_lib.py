"""ctypes binding of libwinoleg_b200.so (include/winoleg_b200.h).

This is the binding a reference maintainer would add; the product API in
``layer.py`` calls only these entry points.  There is no fallback: if the shared library is
missing or fails to load, every call raises.
"""

from __future__ import annotations

import ctypes
import os

from .errors import CudaLayerError, DimensionError

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "libwinoleg_b200.so")

WL_OK, WL_ERR_ARG, WL_ERR_PLAN, WL_ERR_BITS, WL_ERR_CUDA, WL_ERR_WORKSPACE = 0, -1, -2, -3, -4, -5
WL_CANONICAL, WL_LEGENDRE = 0, 1


class wl_qcfg(ctypes.Structure):
    _fields_ = [(n, ctypes.c_int) for n in (
        "input_bits", "weight_bits", "input_transform_bits", "weight_transform_bits",
        "base_change_bits", "hadamard_bits", "output_transform_bits")]


class wl_shape(ctypes.Structure):
    _fields_ = [(n, ctypes.c_int) for n in ("n", "c_in", "c_out", "h", "w", "pad", "images_per_group")]


class wl_stage_stat(ctypes.Structure):
    _fields_ = [("bits", ctypes.c_int), ("max_abs", ctypes.c_double), ("scale", ctypes.c_double)]


_lib = None

EXPORTS = ("wl_plan_create", "wl_plan_destroy", "wl_plan_mode", "wl_weight_cache_size", "wl_weight_transform",
           "wl_weight_transform_f64", "wl_workspace_size", "wl_forward", "wl_forward_f64", "wl_num_stages", "wl_read_stats", "wl_debug_layout",
           "wl_forward_launches", "wl_profile_enable", "wl_profile_read", "wl_backward_workspace_size",
           "wl_backward", "wl_float_workspace_size", "wl_forward_float", "wl_direct_workspace_size",
           "wl_direct_quantized", "wl_direct_quantized_f64", "wl_direct_f64", "wl_train_sizes", "wl_forward_train",
           "wl_debug_set_fix_cap", "wl_debug_gemm_bf16", "wl_last_error")


def lib():
    """Load the library once; raises (no fallback) when it is absent."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        raise CudaLayerError(
            f"{LIB_PATH} is missing: build it with `python -c 'import __graft_entry__ as g; g.build()'` "
            "(nvcc, sm_100a). There is no CPU fallback.")
    L = ctypes.CDLL(LIB_PATH)
    P, I, S, VP = ctypes.POINTER, ctypes.c_int, ctypes.c_size_t, ctypes.c_void_p
    L.wl_plan_create.argtypes = [I, I, I, P(ctypes.c_int64), P(ctypes.c_double), P(VP)]
    L.wl_plan_destroy.argtypes = [VP]
    L.wl_plan_mode.argtypes = [VP]
    L.wl_weight_cache_size.argtypes = [VP, I, I, P(S)]
    L.wl_weight_transform.argtypes = [VP, P(wl_qcfg), VP, I, I, VP, S, VP]
    L.wl_weight_transform_f64.argtypes = [VP, P(wl_qcfg), VP, I, I, VP, S, VP]
    L.wl_workspace_size.argtypes = [VP, P(wl_shape), P(wl_qcfg), P(S)]
    L.wl_forward.argtypes = [VP, P(wl_qcfg), P(wl_shape), VP, VP, VP, VP, VP, S, VP]
    L.wl_forward_f64.argtypes = [VP, P(wl_qcfg), P(wl_shape), VP, VP, VP, VP, VP, S, VP]
    L.wl_train_sizes.argtypes = [VP, P(wl_shape), P(wl_qcfg), P(S), P(S)]
    L.wl_forward_train.argtypes = [VP, P(wl_qcfg), P(wl_shape), VP, VP, VP, VP, VP, S, VP, S, VP]
    L.wl_debug_set_fix_cap.argtypes = [ctypes.c_uint]
    L.wl_debug_gemm_bf16.argtypes = [VP, I, VP, I, I, I, I, I, I, VP, I, ctypes.c_float, VP]
    L.wl_num_stages.argtypes = [VP]
    L.wl_read_stats.argtypes = [VP, P(wl_shape), P(wl_qcfg), VP, VP, P(wl_stage_stat), VP]
    L.wl_debug_layout.argtypes = [VP, P(wl_shape), P(wl_qcfg), P(S), P(I)]
    L.wl_forward_launches.argtypes = [VP, P(wl_shape), P(wl_qcfg)]
    L.wl_backward_workspace_size.argtypes = [VP, P(wl_shape), P(wl_qcfg), P(S)]
    L.wl_backward.argtypes = [VP, P(wl_qcfg), P(wl_shape), VP, VP, VP, VP, VP, VP, VP, S, VP]
    L.wl_float_workspace_size.argtypes = [VP, P(wl_shape), P(S)]
    L.wl_forward_float.argtypes = [VP, P(wl_shape), VP, VP, VP, VP, VP, S, VP]
    L.wl_direct_workspace_size.argtypes = [P(wl_shape), P(S)]
    L.wl_direct_quantized.argtypes = [P(wl_qcfg), P(wl_shape), VP, VP, VP, VP, S, VP]
    L.wl_direct_quantized_f64.argtypes = [P(wl_qcfg), P(wl_shape), VP, VP, VP, VP, S, VP]
    L.wl_direct_f64.argtypes = [P(wl_shape), VP, VP, VP, VP, S, VP]
    L.wl_profile_enable.argtypes = [I]
    L.wl_profile_read.argtypes = [P(ctypes.c_char_p), P(ctypes.c_double), I, P(I), P(I)]
    L.wl_last_error.restype = ctypes.c_char_p
    L.wl_last_error.argtypes = []
    _lib = L
    return L


def check(rc: int, what: str) -> None:
    if rc == WL_OK:
        return
    msg = lib().wl_last_error().decode(errors="replace")
    if rc in (WL_ERR_ARG,):
        raise DimensionError(f"{what}: {msg}")
    if rc in (WL_ERR_BITS, WL_ERR_PLAN):
        raise ValueError(f"{what}: {msg}")
    raise CudaLayerError(f"{what} failed ({rc}): {msg}")


def profile_enable(on: bool) -> None:
    check(lib().wl_profile_enable(int(on)), "wl_profile_enable")


def profile_read() -> tuple[dict, int]:
    """{kernel name: summed ms} over the wl_forward calls since the last read, and the call count."""
    names = (ctypes.c_char_p * 32)()
    ms = (ctypes.c_double * 32)()
    n, calls = ctypes.c_int(), ctypes.c_int()
    check(lib().wl_profile_read(names, ms, 32, ctypes.byref(n), ctypes.byref(calls)), "wl_profile_read")
    return {names[i].decode(): ms[i] for i in range(min(n.value, 32))}, calls.value
