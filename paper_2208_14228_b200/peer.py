"""The G-rank reducer across processes: CUDA IPC peer pointers + stream memory ops.

One process per GPU.  Each rank exports IPC handles of its EST gradient slots,
subtree partial, parameter/velocity replica and two 32-bit signal words, and
maps every peer's.  A step is then (hier.GroupReducer's schedule, per rank):

  phase 1  subtree partial of the rank's own slots        (RankTree(2) only)
  signal   write own sig[0] = step  (cuStreamWriteValue32, ordered after phase 1)
  wait     every peer's sig[0] >= step  (cuStreamWaitValue32 -- the GPU front
           end blocks the stream; no host barrier, no spinning kernel)
  phase 2  owner of shard g: peer LOADS of the G partials (or all E slots for
           owner-computes) over NVLink, fixed rank-order fold, /E and the finite
           check into a staging buffer; the shard's status word is published into
           every rank's gate table (signal / wait sig[2]); then, only if every
           shard of the update was finite, momentum SGD (or Adam) from the staged
           gradients with peer STORES of the updated shard into every replica
           (the reference raises NumericError before it mutates anything,
           model.py:207-209, so a non-finite step leaves every replica as it was)
  signal   own sig[1] = step; wait every peer's sig[1] >= step

so the reduce-scatter, update and parameter all-gather are one kernel per rank
that moves data over NVLink itself, ordered purely on the device.  The control
plane (exchanging handles once) uses torch.distributed (NCCL or gloo).
"""

from __future__ import annotations

import ctypes as C

import torch
import torch.distributed as dist

from . import _native
from .hier import GroupReducer, RankBuffers, _pow2, shard_bounds  # noqa: F401  (shared schedule/shards)
from .device import Flags
from .errors import ConfigError


def _export(t: torch.Tensor) -> tuple[bytes, int]:
    n = _native.lib().bt_ipc_handle_size()
    buf = (C.c_char * n)()
    off = C.c_int64()
    _native.check(_native.lib().bt_ipc_get_handle(t.data_ptr(), buf, C.byref(off)), "ipc export")
    return bytes(buf), off.value


class _Opened:
    """Open each distinct peer allocation once; unmap on close."""

    def __init__(self):
        self.bases: dict[bytes, int] = {}

    def ptr(self, handle: bytes, offset: int) -> int:
        if handle not in self.bases:
            p = C.c_void_p()
            _native.check(_native.lib().bt_ipc_open_handle(handle, C.byref(p)), "ipc open")
            self.bases[handle] = p.value
        return self.bases[handle] + offset

    def close(self):
        for base in self.bases.values():
            _native.lib().bt_ipc_close(base)
        self.bases.clear()


class PeerGroupReducer:
    """This rank's side of a G-rank deterministic reduce over CUDA IPC (see module doc)."""

    NAMES = ("grads", "partial", "param", "vel", "sig", "gate")

    def __init__(self, local: RankBuffers, E: int, variant: str = "rank_tree2", rot: torch.Tensor | None = None,
                 lr: float = 0.02, mu: float = 0.9, group=None, divisor: int = 0, adam: tuple | None = None):
        """E = gradient slots of the job (all ranks); divisor = the mean's denominator (0: E);
        adam = (beta2, eps): Adam update (beta1 = mu, moments in local.vel / local.vel2, bias corrections
        from the step count) instead of momentum SGD."""
        self.group = group
        self.divisor = divisor
        self.adam = adam
        if adam is not None and local.vel2 is None:
            raise ConfigError("Adam needs the second-moment replica (RankBuffers.vel2)")
        if adam is not None:
            self.NAMES = self.NAMES + ("vel2",)
        self.rank, self.G = dist.get_rank(group), dist.get_world_size(group)
        self.local, self.E, self.variant, self.rot, self.lr, self.mu = local, E, variant, rot, lr, mu
        if E % self.G:
            raise ConfigError("E must split into equal contiguous rank blocks")
        self.E_loc = E // self.G
        if variant == "rank_tree2" and not (_pow2(self.E_loc) and _pow2(self.G)):
            raise ConfigError("hierarchical RankTree(2) needs power-of-two E/G and G")
        if variant != "rank_tree2" and E > _native.BT_MAX_TABLE:
            raise ConfigError(f"owner-computes reads at most {_native.BT_MAX_TABLE} slots per element")
        if local.partial is None:
            local.partial = torch.empty_like(local.param)
        self.sig = torch.zeros(3, dtype=torch.int32, device=local.param.device)
        self.gate = torch.zeros(self.G, dtype=torch.int32, device=local.param.device)  # every shard's status
        self.n, self.es = local.param.numel(), local.param.element_size()
        self.dtype = _native.DTYPE_F64 if local.param.dtype == torch.float64 else _native.DTYPE_F32
        self.shards = shard_bounds(self.n, self.G, 16 // self.es)
        lo, hi = self.shards[self.rank]
        self.stage = torch.empty(max(hi - lo, 1), dtype=local.param.dtype, device=local.param.device)
        own = ("sig", "gate")
        mine = {k: _export(getattr(self, k) if k in own else getattr(local, k)) for k in self.NAMES}
        table = [None] * self.G
        dist.all_gather_object(table, mine, group=group)
        self.opened = _Opened()
        self.ptrs = []
        for q in range(self.G):
            if q == self.rank:
                self.ptrs.append({k: (getattr(self, k) if k in own else getattr(local, k)).data_ptr()
                                  for k in self.NAMES})
            else:
                self.ptrs.append({k: self.opened.ptr(*table[q][k]) for k in self.NAMES})
        self.flags = Flags()
        self.step_no = 0

    def _signal_and_wait(self, word: int) -> None:
        s = self.local.stream.cuda_stream
        me = self.ptrs[self.rank]["sig"] + 4 * word
        _native.check(_native.lib().bt_stream_write_u32(me, self.step_no, s), "signal")
        for q in range(self.G):
            if q != self.rank:
                _native.check(_native.lib().bt_stream_wait_u32_geq(self.ptrs[q]["sig"] + 4 * word, self.step_no, s),
                              "wait")

    def step(self) -> None:
        self.step_no += 1
        loc, s = self.local, self.local.stream.cuda_stream
        row = self.n * self.es  # bytes per EST slot row
        if self.variant == "rank_tree2":
            a = _native.ReduceArgs()
            a.dtype, a.mode, a.E, a.fanin, a.n = self.dtype, _native.REDUCE_SUM_ONLY, self.E_loc, 2, self.n
            for k in range(self.E_loc):
                a.grads[k] = loc.grads[k].data_ptr()
            a.param_out = loc.partial.data_ptr()
            _native.check(_native.lib().bt_reduce_update(C.byref(a), s), "subtree")
        self._signal_and_wait(0)
        lo, hi = self.shards[self.rank]
        if hi > lo:
            off = lo * self.es
            a = _native.ReduceArgs()
            a.dtype, a.mode, a.n = self.dtype, _native.REDUCE_UPDATE, hi - lo
            if self.variant == "rank_tree2":
                a.E, a.fanin, a.divisor = self.G, 2, self.divisor or self.E
                for q in range(self.G):
                    a.grads[q] = self.ptrs[q]["partial"] + off
            else:
                a.E, a.fanin, a.divisor = self.E, 0 if self.variant == "sequential" else 2, self.divisor
                for k in range(self.E):
                    a.grads[k] = self.ptrs[k // self.E_loc]["grads"] + (k % self.E_loc) * row + off
                if self.rot is not None:
                    a.rot = self.rot.data_ptr() + lo * 4
            a.param = a.param_out = self.ptrs[self.rank]["param"] + off
            a.vel = a.vel_out = self.ptrs[self.rank]["vel"] + off
            others = [q for q in range(self.G) if q != self.rank]
            a.nout = len(others)
            for i, q in enumerate(others):
                a.extra_param_out[i] = self.ptrs[q]["param"] + off
                a.extra_vel_out[i] = self.ptrs[q]["vel"] + off
            if self.adam is not None:
                b2, eps = self.adam
                a.mode = _native.REDUCE_ADAM
                a.vel2 = a.vel2_out = self.ptrs[self.rank]["vel2"] + off
                for i, q in enumerate(others):
                    a.extra_vel2_out[i] = self.ptrs[q]["vel2"] + off
                a.beta2, a.eps = b2, eps
                a.bc1, a.bc2 = 1.0 / (1.0 - self.mu ** self.step_no), 1.0 / (1.0 - b2 ** self.step_no)
            a.lr, a.mu, a.flags = self.lr, self.mu, self.flags.t.data_ptr()
            # pass 1: fold, /E and the finite check of this shard into the staging buffer
            upd = a.mode
            a.mode, a.param_out, a.stage = _native.REDUCE_MEAN_CHECK, self.stage.data_ptr(), self.stage.data_ptr()
            nout, a.nout = a.nout, 0
            _native.check(_native.lib().bt_reduce_update(C.byref(a), s), "owner check")
            a.mode = _native.REDUCE_APPLY_ADAM if upd == _native.REDUCE_ADAM else _native.REDUCE_APPLY_SGD
            a.param_out, a.nout = a.param, nout
        # publish this shard's status word into every rank's gate table, then wait for every shard's
        for q in range(self.G):
            _native.check(_native.lib().bt_memcpy_async(self.ptrs[q]["gate"] + 4 * self.rank, self.flags.t.data_ptr(),
                                                        4, s), "publish status")
        self._signal_and_wait(2)
        if hi > lo:  # pass 2: the update, only if every shard of the update was finite
            a.gate, a.ngate = self.gate.data_ptr(), self.G
            _native.check(_native.lib().bt_reduce_update(C.byref(a), s), "owner apply")
        self._signal_and_wait(1)

    def check(self) -> None:
        self.flags.raise_if_set("peer group reduce")

    def close(self) -> None:
        torch.cuda.synchronize()
        self.opened.close()
