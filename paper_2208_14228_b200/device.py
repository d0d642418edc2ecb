"""Device plumbing: CUDA tensors as caller-owned memory for the C-ABI.

PyTorch is used only to allocate device memory, get the current stream and
move small host<->device values.  Every computation runs in the sm_100a
library; if no CUDA device is present the calls raise (no CPU fallback).
"""

from __future__ import annotations

import ctypes as C
import struct

import torch

from . import _native

MASK64 = (1 << 64) - 1


def require_cuda() -> torch.device:
    if not torch.cuda.is_available():
        raise RuntimeError("paper_2208_14228_b200 runs on a CUDA device (B200); no CPU fallback exists")
    _native.lib()
    return torch.device("cuda", torch.cuda.current_device())


def stream() -> int:
    return torch.cuda.current_stream().cuda_stream


def f64(*shape) -> torch.Tensor:
    return torch.empty(*shape, dtype=torch.float64, device=require_cuda())


def zeros(*shape, dtype=torch.float64) -> torch.Tensor:
    return torch.zeros(*shape, dtype=dtype, device=require_cuda())


def to_dev(values, dtype=torch.float64) -> torch.Tensor:
    if isinstance(values, torch.Tensor):
        return values.to(device=require_cuda(), dtype=dtype).contiguous()
    return torch.tensor(values, dtype=dtype, device=require_cuda())


def u64_to_i64(x: int) -> int:
    x &= MASK64
    return x - (1 << 64) if x >= (1 << 63) else x


def i64_to_u64(x: int) -> int:
    return int(x) & MASK64


def u64_tensor(values) -> torch.Tensor:
    return torch.tensor([u64_to_i64(v) for v in values], dtype=torch.int64, device=require_cuda())


def ptr(t: torch.Tensor | None) -> int | None:
    return None if t is None else t.data_ptr()


class Flags:
    """The 4-word device status block {status, detail, step, spare}."""

    def __init__(self, t: torch.Tensor | None = None):
        """`t`: an int32[4] device view to hold the words (e.g. the tail of a shard's I/O block)."""
        self.t = torch.zeros(4, dtype=torch.int32, device=require_cuda()) if t is None else t
        self.reset()

    def _stream(self) -> int:  # the current stream of the GPU holding the words
        return torch.cuda.current_stream(self.t.device).cuda_stream

    def reset(self) -> None:
        with torch.cuda.device(self.t.device):
            _native.check(_native.lib().bt_flags_reset(self.t.data_ptr(), self._stream()), "flags reset")

    def status(self) -> tuple[int, int, int]:
        detail, step = C.c_int32(), C.c_int32()
        with torch.cuda.device(self.t.device):
            st = _native.lib().bt_step_status(self.t.data_ptr(), C.byref(detail), C.byref(step), self._stream())
        return st, detail.value, step.value

    def raise_if_set(self, what: str) -> None:
        st, detail, step = self.status()
        if st:
            self.reset()
            exc = _native.STATUS_TO_ERROR.get(st)
            if st == 9 or exc is None:
                raise RuntimeError(f"{what}: device failure (status {st}) {_native.last_error()}")
            if st == 5:
                raise exc(f"{what}: non-finite synchronized gradient at parameter {detail} (step {step})")
            if st == 6:
                raise exc(f"{what}: executor replica diverged (replica {detail})")
            raise exc(f"{what}: status {st}")


class DeviceVector:
    """List-like view of a 1-D float64 device tensor (lazy D2H on read).

    The reference exposes parameters, velocities and gradients as Python lists
    (model.py:44-85); this view keeps that surface (len, index, slice,
    iteration, == against lists) while the data stays in HBM.  Item
    assignment writes through to the device.
    """

    __slots__ = ("t",)

    def __init__(self, t: torch.Tensor):
        self.t = t

    def tolist(self) -> list[float]:
        return self.t.tolist()

    def __len__(self) -> int:
        return self.t.numel()

    def __iter__(self):
        return iter(self.tolist())

    def __getitem__(self, i):
        if isinstance(i, slice):
            return self.tolist()[i]
        return float(self.t[i].item())

    def __setitem__(self, i, v) -> None:
        self.t[i] = float(v)

    def __eq__(self, other) -> bool:
        if isinstance(other, DeviceVector):
            other = other.tolist()
        try:
            return self.tolist() == list(other)
        except TypeError:
            return NotImplemented

    def __ne__(self, other) -> bool:
        eq = self.__eq__(other)
        return eq if eq is NotImplemented else not eq

    __hash__ = None

    def __repr__(self) -> str:
        return f"DeviceVector({self.tolist()!r})"

    def to_bytes(self) -> bytes:
        return self.t.detach().to("cpu").numpy().astype("<f8").tobytes()


def floats_to_bytes(values) -> bytes:
    if isinstance(values, DeviceVector):
        return values.to_bytes()
    if isinstance(values, torch.Tensor):
        return values.detach().to("cpu").numpy().astype("<f8").tobytes()
    return struct.pack(f"<{len(values)}d", *values)
