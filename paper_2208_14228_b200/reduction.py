"""Reduction shapes (reduction.py:20-84 of the reference) and reduce_sum.

`Sequential` is a strict left fold from the first element; `Tree(f)` is the
bottom-up f-ary tree with children folded left to right.  The shape is part
of the contract: every sm_100a kernel in this package folds in exactly the
shape named here, keyed by EST rank.
"""

from __future__ import annotations

from dataclasses import dataclass

import torch

from . import _native
from .device import ptr, require_cuda, stream, to_dev


@dataclass(frozen=True)
class Sequential:
    """Left-to-right fold; identical on every device kind."""


@dataclass(frozen=True)
class Tree:
    """Bottom-up tree of the given fanin (a device-kind surrogate)."""

    fanin: int

    def __post_init__(self):
        if self.fanin < 1:
            raise ValueError(f"fanin must be positive, got {self.fanin}")


ReduceVariant = Sequential | Tree


def fanin_code(variant: ReduceVariant) -> int:
    """C-ABI encoding: 0 = Sequential, f >= 2 = Tree(f).  Tree(1) never
    terminates in the reference (its level loop cannot shrink); rejected."""
    if isinstance(variant, Sequential):
        return 0
    if isinstance(variant, Tree):
        if variant.fanin == 1:
            from .errors import ConfigError

            raise ConfigError("Tree(1) cannot reduce (the reference loops forever); use fanin >= 2")
        return variant.fanin
    raise TypeError(f"not a reduction variant: {variant!r}")


def reduce_sum(values, variant: ReduceVariant) -> float:
    """Sum under the given shape on the device (empty -> 0.0)."""
    require_cuda()
    v = to_dev(values) if not isinstance(values, torch.Tensor) else values.to(torch.float64).contiguous()
    out = torch.zeros(1, dtype=torch.float64, device="cuda")
    _native.check(_native.lib().bt_reduce_sum_f64(ptr(v) if v.numel() else None, v.numel(), fanin_code(variant),
                                                  ptr(out), stream()))
    return float(out.item())


@dataclass(frozen=True)
class KernelProfile:
    """Reduction behaviour of one device kind (reduction.py:65-84)."""

    device_kind: str
    reduce_variant: ReduceVariant

    @classmethod
    def native(cls, device_kind: str, fanin: int) -> "KernelProfile":
        return cls(device_kind, Tree(fanin))

    @classmethod
    def device_agnostic(cls, device_kind: str) -> "KernelProfile":
        return cls(device_kind, Sequential())
