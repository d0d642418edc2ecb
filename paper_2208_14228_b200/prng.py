"""splitmix64 primitives (the reference's prng.py:27-93 API).

The scalar, inherently sequential entry points (one draw, a Fisher-Yates
chain, a byte-serial hash) run in the native host half of the C-ABI; bulk
draws used by the step run on the device in counter form
(`draws`, draw n of state s0 = mix64(s0 + (n+1)*gamma)).
"""

from __future__ import annotations

import ctypes as C

import numpy as np
import torch

from . import _native
from .device import ptr, require_cuda, stream

MASK64 = (1 << 64) - 1
GOLDEN_GAMMA = 0x9E3779B97F4A7C15  # prng.py:14
TAG_DATASET = 0xD5A61C0FFEE5EED5  # prng.py:20-24
TAG_MODEL_INIT = 0x1417E5EED0D0CAFE
TAG_DROPOUT = 0xD80F0D7A6B15EA5E
TAG_DATA_WORKER = 0xB07C9E11A7756E1D
TAG_BUCKET_ARRIVAL = 0xAC1DB0B5CA77E7E5


def mix64(x: int) -> int:
    return _native.lib().bt_host_mix64(x & MASK64)


def splitmix64_next(state: int) -> tuple[int, int]:
    """(state + gamma, mix64(state + gamma))  -- prng.py:38-45."""
    state = (state + GOLDEN_GAMMA) & MASK64
    return state, mix64(state)


def unit_float(raw: int) -> float:
    return (raw >> 11) * 2.0**-53  # exact: a 53-bit integer times a power of two


def rng_uniform01(state: int) -> tuple[int, float]:
    state, raw = splitmix64_next(state)
    return state, unit_float(raw)


def derive_stream(*words: int) -> int:
    return _native.host_derive_stream(*words)


def fnv1a64(data: bytes) -> int:
    return _native.host_fnv1a64(bytes(data))


def shuffled_range(n: int, state: int) -> list[int]:
    out = np.zeros(max(n, 1), dtype=np.int32)
    _native.check(_native.lib().bt_host_shuffled_range(n, state & MASK64, out.ctypes.data_as(C.POINTER(C.c_int32))))
    return out[:n].tolist()


def draws(state: int, first: int, n: int) -> tuple[torch.Tensor, torch.Tensor]:
    """Device: raw words and uniforms of draws [first, first+n) of a stream."""
    require_cuda()
    raw = torch.empty(n, dtype=torch.int64, device="cuda")
    uni = torch.empty(n, dtype=torch.float64, device="cuda")
    _native.check(_native.lib().bt_splitmix64_draws(state & MASK64, first, n, ptr(raw), ptr(uni), stream()))
    return raw, uni
