"""Bucket maps and the deterministic allreduce (reference buckets.py:1-124).

The bucket map is host metadata; the combine runs in the sm_100a reducer
(bt_reduce.cu).  Under a Tree kernel the reference starts each parameter's
rank cycle at its ring chunk, start = pos*nrep//len(bucket)
(buckets.py:119-122); that start is precomputed per parameter
(`rotation_table`) and handed to the device, so the device fold order is
exactly the reference's.
"""

from __future__ import annotations

import ctypes as C
from dataclasses import dataclass

import numpy as np
import torch

from . import _native
from .device import DeviceVector, ptr, require_cuda, stream, to_dev
from .errors import InputError
from .prng import fnv1a64
from .reduction import ReduceVariant, Sequential, fanin_code

_i32p = C.POINTER(C.c_int32)


@dataclass(frozen=True)
class BucketMap:
    """Ordered partition of [0, param_count) into ordered buckets."""

    capacity: int
    buckets: tuple[tuple[int, ...], ...]

    @property
    def param_count(self) -> int:
        return sum(len(b) for b in self.buckets)

    def covered_exactly_once(self) -> bool:
        flat = [i for b in self.buckets for i in b]
        return sorted(flat) == list(range(len(flat)))


def _pack(order: list[int], capacity: int) -> BucketMap:
    return BucketMap(capacity, tuple(tuple(order[i:i + capacity]) for i in range(0, len(order), capacity)))


def build_buckets_initial(param_count: int, capacity: int) -> BucketMap:
    """Descending parameter index packed greedily (buckets.py:47-53)."""
    if capacity < 1:
        raise InputError(f"bucket capacity must be >= 1, got {capacity}")
    return _pack(list(range(param_count - 1, -1, -1)), capacity)


def rebuild_buckets_first_minibatch(arrival_perm: list[int], capacity: int) -> BucketMap:
    """Repack in arrival order (buckets.py:56-60)."""
    if sorted(arrival_perm) != list(range(len(arrival_perm))):
        raise InputError("arrival order is not a permutation of the parameter indices")
    return _pack(list(arrival_perm), capacity)


def layout_arrival_perm(param_count: int, layout_key: list[tuple[str, int]]) -> list[int]:
    """Layout-keyed arrival order (buckets.py:70-82), native host Fisher-Yates."""
    n = len(layout_key)
    kinds = (C.c_uint64 * max(n, 1))(*[fnv1a64(k.encode("utf-8")) for k, _ in layout_key])
    threads = (C.c_int64 * max(n, 1))(*[t for _, t in layout_key])
    perm = np.zeros(max(param_count, 1), dtype=np.int32)
    _native.check(_native.lib().bt_host_layout_arrival_perm(param_count, n, kinds, threads,
                                                            perm.ctypes.data_as(_i32p)))
    return perm[:param_count].tolist()


def rotation_table(bucket_map: BucketMap, nrep: int) -> np.ndarray:
    """Per-parameter rank-cycle start pos*nrep//len(bucket) (buckets.py:119-122)."""
    n = bucket_map.param_count
    sizes = np.array([len(b) for b in bucket_map.buckets], dtype=np.int32)
    idx = np.array([i for b in bucket_map.buckets for i in b], dtype=np.int32)
    rot = np.zeros(max(n, 1), dtype=np.int32)
    _native.check(_native.lib().bt_host_rotation_table(len(sizes), sizes.ctypes.data_as(_i32p),
                                                       idx.ctypes.data_as(_i32p), nrep, n, rot.ctypes.data_as(_i32p)))
    return rot[:n]


def _replica_tensor(rep) -> torch.Tensor:
    if isinstance(rep, DeviceVector):
        return rep.t
    if isinstance(rep, torch.Tensor):
        return rep.to(device="cuda", dtype=torch.float64).contiguous()
    return to_dev(list(rep))


def allreduce(replicas, bucket_map: BucketMap, variant: ReduceVariant) -> list[float]:
    """Synchronized mean of rank-ordered gradient replicas (buckets.py:85-124).

    Runs the device reducer in MEAN_ONLY mode.  ``replicas`` is ordered by
    ascending virtual rank; each may be a list, a DeviceVector or a tensor.
    """
    if not replicas:
        raise InputError("need at least one gradient replica")
    require_cuda()
    reps = [_replica_tensor(r) for r in replicas]
    nparams = reps[0].numel()
    if any(r.numel() != nparams for r in reps):
        raise InputError("gradient replicas have mismatched lengths")
    if bucket_map.param_count != nparams:
        raise InputError(f"bucket map covers {bucket_map.param_count} parameters, replicas have {nparams}")
    return allreduce_device(reps, bucket_map, variant).tolist()


def allreduce_device(reps: list[torch.Tensor], bucket_map: BucketMap, variant: ReduceVariant) -> torch.Tensor:
    """Device result of allreduce (no host copy)."""
    nrep, nparams = len(reps), reps[0].numel()
    fan = fanin_code(variant)
    out = torch.empty(nparams, dtype=torch.float64, device="cuda")
    a = _native.ReduceArgs()
    a.dtype, a.mode, a.E, a.fanin, a.n = _native.DTYPE_F64, _native.REDUCE_MEAN_ONLY, nrep, fan, nparams
    keep = []
    if nrep <= _native.BT_MAX_TABLE:
        for k, r in enumerate(reps):
            a.grads[k] = ptr(r)
    else:
        stacked = torch.stack(reps)
        keep.append(stacked)
        a.grads[0] = ptr(stacked)
        a.grads_ld = nparams
    rot = None
    if not isinstance(variant, Sequential):
        rot = torch.from_numpy(rotation_table(bucket_map, nrep)).to("cuda")
        a.rot = ptr(rot)
    a.param_out = ptr(out)
    _native.check(_native.lib().bt_reduce_update(C.byref(a), stream()), "allreduce")
    return out
