"""TEST INFRASTRUCTURE ONLY — Python face of the C oracle (``liboracle.so``).

Mirrors the reference API so parity tests read like the reference's own tests:

* ``fake_quant(x, bits)``                          reference quantize.py:112-126
* ``compute_scale(x, bits)``                       quantize.py:103-109
* ``conv2d_winograd_quantized(x, w, mode, bits)``  quantize.py:129-148 for one image [c_in,H,W]
* ``quant_conv_batch(x, w, mode, bits, padding, images_per_group)``: the batched extension the
  B200 layer implements (stage scales shared by ``images_per_group`` images; 1 == per-image,
  i.e. exactly N independent reference calls).

Only tests/, bench.py's cpu-baseline leg and __graft_entry__.smoke may import this module; the
product package never does.
"""

from __future__ import annotations

import ctypes
import os
import subprocess
from dataclasses import dataclass

import numpy as np

from . import plan_ref

_HERE = os.path.dirname(os.path.abspath(__file__))
_LIB = None

STAGES = {
    "canonical": ("input", "weights", "weight_transform", "input_transform", "hadamard", "output"),
    "legendre": ("input", "weights", "weight_transform", "weight_base_change", "input_base_change",
                 "input_transform", "hadamard", "output_base_change", "output"),
}
# order of the 7 widths handed to C: input, weights, input_transform, weight_transform, base_change,
# hadamard, output  (reference quantize.py:40-55 field names)
BIT_FIELDS = ("input_bits", "weight_bits", "input_transform_bits", "weight_transform_bits",
              "base_change_bits", "hadamard_bits", "output_transform_bits")
STAGE_BIT_FIELD = {
    "input": "input_bits", "weights": "weight_bits", "weight_transform": "weight_transform_bits",
    "weight_base_change": "base_change_bits", "input_base_change": "base_change_bits",
    "input_transform": "input_transform_bits", "hadamard": "hadamard_bits",
    "output_base_change": "base_change_bits", "output": "output_transform_bits",
}


def build() -> str:
    path = os.path.join(_HERE, "liboracle.so")
    src = os.path.join(_HERE, "winoleg_oracle.c")
    if not os.path.exists(path) or os.path.getmtime(path) < os.path.getmtime(src):
        subprocess.run(["make", "-s", "-C", _HERE], check=True)
    return path


def lib():
    global _LIB
    if _LIB is None:
        _LIB = ctypes.CDLL(build())
        _LIB.wlo_quant_conv.restype = ctypes.c_int
        _LIB.wlo_fake_quant.restype = ctypes.c_double
    return _LIB


@dataclass(frozen=True)
class Stat:
    stage: str
    bits: int
    max_abs: float
    scale: float


def _bits_array(bits: dict) -> np.ndarray:
    return np.array([int(bits[f]) for f in BIT_FIELDS], dtype=np.int32)


def uniform_bits(b: int, hadamard: int | None = None) -> dict:
    d = {f: b for f in BIT_FIELDS}
    if hadamard is not None:
        d["hadamard_bits"] = hadamard
    return d


def _ptr(a: np.ndarray, ctype=ctypes.c_double):
    return a.ctypes.data_as(ctypes.POINTER(ctype))


def fake_quant(x, bits: int):
    a = np.array(x, dtype=np.float64, copy=True).ravel()
    s = ctypes.c_double()
    lib().wlo_fake_quant(_ptr(a), ctypes.c_long(a.size), ctypes.c_int(bits), ctypes.byref(s), None)
    return a.reshape(np.shape(x))


def fake_quant_codes(x, bits: int):
    a = np.array(x, dtype=np.float64, copy=True).ravel()
    codes = np.zeros(a.size, dtype=np.int32)
    s = ctypes.c_double()
    mx = lib().wlo_fake_quant(_ptr(a), ctypes.c_long(a.size), ctypes.c_int(bits), ctypes.byref(s),
                              _ptr(codes, ctypes.c_int32))
    return codes.reshape(np.shape(x)), float(mx), float(s.value)


def quant_conv_batch(x, w, mode: str, bits: dict, padding: int = 0, images_per_group: int = 1,
                     capture: bool = False, nthreads: int | None = None, identity_base: bool = False):
    """x [n,c_in,H,W], w [c_out,c_in,3,3] -> (y [n,c_out,Ho,Wo] fp64, stats[groups][stages], codes|None)."""
    x = np.asarray(x, dtype=np.float64)
    w = np.ascontiguousarray(w, dtype=np.float64)
    if padding:
        x = np.pad(x, ((0, 0), (0, 0), (padding, padding), (padding, padding)))
    x = np.ascontiguousarray(x)
    n, cin, h, wd = x.shape
    cout, _, k, _ = w.shape
    o = 4
    m = o + k - 1
    leg = mode == "legendre"
    mats = plan_ref.packed_f64(o, k, identity_base=identity_base)
    oh, ow = h - k + 1, wd - k + 1
    th, tw = -(-oh // o), -(-ow // o)
    T = th * tw
    y = np.zeros((n, cout, oh, ow))
    ngroups = n // images_per_group
    stats = np.zeros((ngroups, 9, 3))
    names = STAGES[mode]
    cap_arrays = None
    cap_ptrs = None
    if capture:
        shapes = {
            "input": (n, cin, h, wd), "weights": (cout, cin, k, k),
            "weight_transform": (cout, cin, m, m), "weight_base_change": (cout, cin, m, m),
            "input_base_change": (n, cin, T, m, m), "input_transform": (n, cin, T, m, m),
            "hadamard": (n, cout, T, m, m), "output_base_change": (n, cout, T, m, m),
            "output": (n, cout, oh, ow),
        }
        cap_arrays = {s: np.zeros(shapes[s], dtype=np.int32) for s in names}
        cap_ptrs = (ctypes.POINTER(ctypes.c_int32) * 9)()
        for i, s in enumerate(names):
            cap_ptrs[i] = _ptr(cap_arrays[s], ctypes.c_int32)
    if nthreads is None:
        nthreads = os.cpu_count() or 1
    rc = lib().wlo_quant_conv(
        _ptr(x), n, cin, h, wd, _ptr(w), cout, _ptr(mats), o, k, int(leg),
        _ptr(_bits_array(bits), ctypes.c_int), images_per_group, _ptr(y), _ptr(stats),
        cap_ptrs, nthreads)
    if rc != 0:
        raise ValueError(f"oracle rejected the call (rc={rc})")
    st = [[Stat(names[i], int(stats[g, i, 0]), float(stats[g, i, 1]), float(stats[g, i, 2]))
           for i in range(len(names))] for g in range(ngroups)]
    return y, st, cap_arrays


def conv2d_winograd_quantized(x, w, mode: str, bits: dict, identity_base: bool = False):
    """One reference call: x [c_in,H,W] (no padding added) -> (y [c_out,Ho,Wo], [Stat...])."""
    y, st, _ = quant_conv_batch(np.asarray(x)[None], w, mode, bits, 0, 1, nthreads=1,
                                identity_base=identity_base)
    return y[0], st[0]
