"""Executors onto GPUs: the EST->GPU mapper of the north star.

The reference places a layout's executors as Python objects (engine.py:169-199, 202-243); here
one process drives every GPU of the box and executor x of a layout runs on a CUDA device:

  * the devices are `devices()` -- every visible GPU, or the list given to `set_devices`
    (a list may repeat an ordinal: several logical devices on one GPU, which is how the
    multi-device paths are exercised on a one-GPU machine);
  * executors map to devices in contiguous, balanced blocks (`executor_devices`), so the ESTs
    of a device are one contiguous rank block (assign_ranks keeps executors contiguous) -- the
    shape the hierarchical RankTree(2) reduction and the lock-step exchange need;
  * peer access is enabled between every pair of distinct GPUs in use, so kernels on one GPU
    load and store the others' memory over NVLink.

`XGroup` holds the per-device exchange buffers of a lock-step multi-device step (bt_mlp.cu,
n_dev > 1): a slot inbox of [2][E][BT_XSP] values per device, 16 bytes per value (two tagged
8-byte words).
"""

from __future__ import annotations

import torch

from . import _native
from .errors import ConfigError

_devices: list[int] | None = None
_peer_done: set[tuple[int, int]] = set()


def set_devices(devices: list[int] | None) -> None:
    """Devices the engine places executors on (None: every visible GPU).  Takes effect for the
    next init_training / apply_layout / checkpoint_restore."""
    global _devices
    if devices is not None:
        devices = [int(d) for d in devices]
        n = torch.cuda.device_count()
        if not devices or any(d < 0 or d >= n for d in devices):
            raise ConfigError(f"devices {devices} outside the {n} visible GPUs")
        if len(devices) > _native.BT_MAX_XDEV:
            raise ConfigError(f"at most {_native.BT_MAX_XDEV} devices per job")
    _devices = devices


def devices() -> list[int]:
    if _devices is not None:
        return list(_devices)
    n = torch.cuda.device_count()
    return list(range(min(max(n, 1), _native.BT_MAX_XDEV)))


def executor_devices(n_exec: int, devs: list[int] | None = None) -> list[int]:
    """Logical device index of every executor: contiguous balanced blocks over min(X, D) devices."""
    devs = devices() if devs is None else devs
    n = min(n_exec, len(devs))
    return [x * n // n_exec for x in range(n_exec)]


def enable_peer_access(ordinals: list[int]) -> None:
    """cudaDeviceEnablePeerAccess between every ordered pair of distinct GPUs (once per process)."""
    uniq = sorted(set(ordinals))
    for d in uniq:
        for p in uniq:
            if d != p and (d, p) not in _peer_done:
                with torch.cuda.device(d):
                    _native.check(_native.lib().bt_enable_peer_access(p), f"peer access {d}->{p}")
                _peer_done.add((d, p))


class XGroup:
    """Exchange buffers of one lock-step multi-device step: one zero-initialised inbox per device."""

    def __init__(self, ordinals: list[int], E: int):
        self.ordinals, self.E = list(ordinals), E
        self.inbox = []
        for d in self.ordinals:
            with torch.cuda.device(d):
                self.inbox.append(torch.zeros(inbox_words(E), dtype=torch.int64, device="cuda"))

    def table(self) -> list[int]:
        return [t.data_ptr() for t in self.inbox]


def inbox_words(E: int) -> int:
    """8-byte words of one device's inbox: [2 parities][E][BT_XSP][2 tagged halves]."""
    return 2 * E * _native.BT_XSP * 2


__all__ = ["set_devices", "devices", "executor_devices", "enable_peer_access", "XGroup", "inbox_words"]
