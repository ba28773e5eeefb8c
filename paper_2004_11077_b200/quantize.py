"""Quantization configuration types, with the reference's names and validation
(reference quantize.py:21-100).  The arithmetic itself runs on the GPU (layer.py -> C ABI)."""

from __future__ import annotations

from dataclasses import dataclass, fields


@dataclass(frozen=True)
class QuantParams:
    """Per-tensor symmetric quantization parameters (quantize.py:21-37)."""

    bits: int
    scale: float
    rounding: str = "half-even"

    def __post_init__(self):
        if self.bits < 2:
            raise ValueError(f"need at least 2 bits, got {self.bits}")
        if not self.scale > 0:
            raise ValueError(f"scale must be positive, got {self.scale}")

    @property
    def q_max(self) -> int:
        return 2 ** (self.bits - 1) - 1


@dataclass(frozen=True)
class QuantConfig:
    """Bit width of every stage boundary (quantize.py:40-76)."""

    input_bits: int = 8
    weight_bits: int = 8
    input_transform_bits: int = 8
    weight_transform_bits: int = 8
    base_change_bits: int = 8
    hadamard_bits: int = 8
    output_transform_bits: int = 8

    def __post_init__(self):
        for f in fields(self):
            if getattr(self, f.name) < 2:
                raise ValueError(f"{f.name} must be >= 2, got {getattr(self, f.name)}")

    @classmethod
    def uniform(cls, bits: int, hadamard_bits: int | None = None) -> "QuantConfig":
        h = bits if hadamard_bits is None else hadamard_bits
        return cls(bits, bits, bits, bits, bits, h, bits)

    @classmethod
    def from_name(cls, name: str) -> "QuantConfig":
        """"8b" (uniform) or "8b+9b" (wider Hadamard stage)."""
        parts = name.strip().lower().split("+")
        try:
            widths = [int(p.removesuffix("b")) for p in parts]
        except ValueError:
            widths = []
        if len(widths) == 1:
            return cls.uniform(widths[0])
        if len(widths) == 2:
            return cls.uniform(widths[0], hadamard_bits=widths[1])
        raise ValueError(f"cannot parse quantization config name {name!r}")

    def as_tuple(self) -> tuple[int, ...]:
        return tuple(getattr(self, f.name) for f in fields(self))


# stage name -> QuantConfig field (quantize.py:80-90)
STAGE_BITS = {
    "input": "input_bits",
    "weights": "weight_bits",
    "weight_transform": "weight_transform_bits",
    "weight_base_change": "base_change_bits",
    "input_base_change": "base_change_bits",
    "input_transform": "input_transform_bits",
    "hadamard": "hadamard_bits",
    "output_base_change": "base_change_bits",
    "output": "output_transform_bits",
}

STAGE_ORDER = {
    "canonical": ("input", "weights", "weight_transform", "input_transform", "hadamard", "output"),
    "legendre": ("input", "weights", "weight_transform", "weight_base_change", "input_base_change",
                 "input_transform", "hadamard", "output_base_change", "output"),
}


@dataclass(frozen=True)
class StageStat:
    """Observed range and scale of one stage cast (quantize.py:93-100)."""

    stage: str
    bits: int
    max_abs: float
    scale: float
