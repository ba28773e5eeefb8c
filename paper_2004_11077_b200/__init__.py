"""B200-native quantized Winograd F(4x4,3x3) layer, canonical or monic-Legendre base.

A from-scratch sm_100a implementation of the hot path of the reference ``winoleg`` package
(arXiv 2004.11077): host construction of the transforms (plan.py), a C-ABI shared library of
hand-written CUDA kernels (csrc/, include/winoleg_b200.h) and a PyTorch-facing API (layer.py).
"""

from .errors import CudaLayerError, DimensionError, InvalidPointsError
from .layer import (BASE_MODES, QuantWinogradConv, WinogradAwareConv2d, conv2d_direct, conv2d_direct_quantized,
                    conv2d_winograd,
                    conv2d_winograd_quantized,
                    default_plan, winograd_conv2d)
from .plan import (BaseChange, InterpolationPoints, Rational, WinogradPlan, build_base_change, build_plan,
                   monic_legendre, plan_to_float, poly_from_roots, stage_matrices)
from .quantize import STAGE_BITS, STAGE_ORDER, QuantConfig, QuantParams, StageStat

__version__ = "0.1.0"

__all__ = [
    "BASE_MODES", "QuantWinogradConv", "WinogradAwareConv2d", "conv2d_direct", "conv2d_direct_quantized",
    "conv2d_winograd",
    "conv2d_winograd_quantized",
    "default_plan",
    "winograd_conv2d",
    "BaseChange", "InterpolationPoints", "Rational", "WinogradPlan", "build_base_change", "build_plan",
    "monic_legendre", "plan_to_float", "poly_from_roots", "stage_matrices",
    "STAGE_BITS", "STAGE_ORDER", "QuantConfig", "QuantParams", "StageStat",
    "CudaLayerError", "DimensionError", "InvalidPointsError", "__version__",
]
