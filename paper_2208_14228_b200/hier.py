"""The G-GPU deterministic reducer: hierarchical RankTree(2) and owner-computes.

Every rank g holds the EST slots of its contiguous rank block (E/G slots of n
elements), a parameter/velocity replica, and a stream.  A reduction step is two
stream-ordered phases, synchronised only by CUDA events (no host barrier, no
device spin -- nothing can deadlock):

  RankTree(2) (the B200 default, E/G and G powers of two):
    1. each rank folds its own slots into a partial (BT_REDUCE_SUM_ONLY) --
       the complete binary subtree of its contiguous rank block;
    2. the owner of parameter shard s folds the G partials of s in rank order
       (the top log2(G) levels of the same tree), divides by E, applies
       momentum SGD, and stores the updated shard into EVERY rank's replica
       (peer stores: the parameter all-gather fused into the same pass).
    The association is exactly the flat Tree(2) over all E slots, so weights
    are bit-identical to the single-GPU reducer (tests/test_gpu_hier.py).
    NVLink bytes per GPU: (G-1)/G*S in (partials) + (G-1)/G*S out (params).

  Owner-computes (Sequential, or Tree with the reference's ring rotation):
    the shard owner reads all E slots of its shard directly (peer loads in
    rank order, rotation per parameter) and folds them exactly like one GPU.
    NVLink bytes per GPU: (G-1)*E*S/G^2 in + (G-1)/G*S out.

The buffers of other ranks are addressed by raw device pointers: in one
process driving several GPUs (peer access enabled), in one GPU simulating G
ranks (the tests), or across processes through CUDA IPC handles
(bt_ipc_get_handle / bt_ipc_open_handle) -- the kernels do not care.
"""

from __future__ import annotations

import ctypes as C
from dataclasses import dataclass

import torch

from . import _native
from .device import Flags
from .errors import ConfigError


@dataclass
class RankBuffers:
    grads: torch.Tensor    # [E/G, n] this rank's EST gradient slots (ascending virtual rank)
    param: torch.Tensor    # [n] replica
    vel: torch.Tensor      # [n] replica
    stream: torch.cuda.Stream
    partial: torch.Tensor | None = None  # [n] RankTree subtree sum
    vel2: torch.Tensor | None = None     # [n] Adam second moment (replica), when the update is Adam


def shard_bounds(n: int, G: int, align: int = 4) -> list[tuple[int, int]]:
    """Contiguous parameter shards, boundaries multiples of `align` elements (16-byte vectors)."""
    units = -(-n // align)
    base, extra = divmod(units, G)
    out, start = [], 0
    for g in range(G):
        u = base + (1 if g < extra else 0)
        lo, hi = min(start * align, n), min((start + u) * align, n)
        out.append((lo, hi))
        start += u
    return out


def _pow2(x: int) -> bool:
    return x > 0 and (x & (x - 1)) == 0


class GroupReducer:
    """One deterministic reduce + SGD over G ranks' EST slots (see module doc)."""

    def __init__(self, ranks: list[RankBuffers], E: int, variant: str = "rank_tree2", rot: torch.Tensor | None = None,
                 lr: float = 0.02, mu: float = 0.9):
        self.ranks, self.G, self.E = ranks, len(ranks), E
        if E % self.G:
            raise ConfigError("E must split into equal contiguous rank blocks")
        self.E_loc = E // self.G
        self.n = ranks[0].param.numel()
        self.dtype = ranks[0].param.dtype
        self.variant, self.rot, self.lr, self.mu = variant, rot, lr, mu
        if variant == "rank_tree2" and not (_pow2(self.E_loc) and _pow2(self.G)):
            raise ConfigError("hierarchical RankTree(2) needs power-of-two E/G and G (use owner-computes)")
        if variant != "rank_tree2" and E > _native.BT_MAX_TABLE:
            raise ConfigError(f"owner-computes reads at most {_native.BT_MAX_TABLE} slots per element")
        if self.G - 1 > _native.BT_MAX_REPLICA_OUT:
            raise ConfigError("at most 9 ranks per group")
        if variant == "rank_tree2":
            for r in ranks:
                if r.partial is None:
                    r.partial = torch.empty_like(r.param)
        self.shards = shard_bounds(self.n, self.G, 16 // ranks[0].param.element_size())
        self.flags = []
        self.stage, self.gate = [], []
        for r, (lo, hi) in zip(ranks, self.shards):  # per rank: status, staged shard gradients, gate table
            with torch.cuda.device(r.param.device):
                self.flags.append(Flags())
                self.stage.append(torch.empty(max(hi - lo, 1), dtype=r.param.dtype, device=r.param.device))
                self.gate.append(torch.zeros(self.G, dtype=torch.int32, device=r.param.device))
        self.es = ranks[0].param.element_size()

    def _dtype_code(self) -> int:
        return _native.DTYPE_F64 if self.dtype == torch.float64 else _native.DTYPE_F32

    def step(self) -> None:
        G, n = self.G, self.n
        ev1 = []
        if self.variant == "rank_tree2":  # phase 1: per-rank subtree partials
            for r in self.ranks:
                with torch.cuda.stream(r.stream):
                    a = _native.ReduceArgs()
                    a.dtype, a.mode, a.E, a.fanin, a.n = self._dtype_code(), _native.REDUCE_SUM_ONLY, self.E_loc, 2, n
                    for k in range(self.E_loc):
                        a.grads[k] = r.grads[k].data_ptr()
                    a.param_out = r.partial.data_ptr()
                    _native.check(_native.lib().bt_reduce_update(C.byref(a), r.stream.cuda_stream), "subtree")
                    e = torch.cuda.Event()
                    e.record(r.stream)
                    ev1.append(e)
        evp, pending = [], []
        for g, r in enumerate(self.ranks):  # phase 2: shard owners
            lo, hi = self.shards[g]
            with torch.cuda.stream(r.stream):
                for e in ev1:
                    r.stream.wait_event(e)
                if hi > lo:
                    a = _native.ReduceArgs()
                    a.dtype, a.mode, a.n = self._dtype_code(), _native.REDUCE_UPDATE, hi - lo
                    off = lo * self.es
                    if self.variant == "rank_tree2":
                        a.E, a.fanin, a.divisor = G, 2, self.E
                        for q, rq in enumerate(self.ranks):
                            a.grads[q] = rq.partial.data_ptr() + off
                    else:
                        a.E, a.fanin = self.E, 0 if self.variant == "sequential" else 2
                        for k in range(self.E):
                            a.grads[k] = self.ranks[k // self.E_loc].grads[k % self.E_loc].data_ptr() + off
                        if self.rot is not None:
                            a.rot = self.rot.data_ptr() + lo * 4
                    a.param, a.vel = r.param.data_ptr() + off, r.vel.data_ptr() + off
                    a.param_out, a.vel_out = a.param, a.vel
                    others = [q for q in range(G) if q != g]
                    a.nout = len(others)
                    for i, q in enumerate(others):  # the all-gather: peer stores of the updated shard
                        a.extra_param_out[i] = self.ranks[q].param.data_ptr() + off
                        a.extra_vel_out[i] = self.ranks[q].vel.data_ptr() + off
                    a.lr, a.mu, a.flags = self.lr, self.mu, self.flags[g].t.data_ptr()
                    # pass 1: fold, /E, finite check of the shard into the staging buffer
                    a.mode, a.param_out, a.stage = _native.REDUCE_MEAN_CHECK, self.stage[g].data_ptr(), self.stage[g].data_ptr()
                    nout, a.nout = a.nout, 0
                    _native.check(_native.lib().bt_reduce_update(C.byref(a), r.stream.cuda_stream), "owner check")
                    a.mode, a.param_out, a.nout = _native.REDUCE_APPLY_SGD, a.param, nout
                    a.gate, a.ngate = self.gate[g].data_ptr(), G
                    pending.append((g, a))
                for q in range(G):  # publish the shard's status word into every rank's gate table
                    _native.check(_native.lib().bt_memcpy_async(self.gate[q].data_ptr() + 4 * g,
                                                                self.flags[g].t.data_ptr(), 4, r.stream.cuda_stream),
                                  "publish status")
                e = torch.cuda.Event()
                e.record(r.stream)
                evp.append(e)
        for g, a in pending:  # pass 2: the update, only if every shard was finite
            r = self.ranks[g]
            with torch.cuda.stream(r.stream):
                for e in evp:
                    r.stream.wait_event(e)
                _native.check(_native.lib().bt_reduce_update(C.byref(a), r.stream.cuda_stream), "owner apply")
        ev2 = []
        for r in self.ranks:
            e = torch.cuda.Event()
            e.record(r.stream)
            ev2.append(e)
        for r in self.ranks:  # every replica complete before a rank's next kernels
            for e in ev2 + evp:
                r.stream.wait_event(e)

    def check(self) -> None:
        for f in self.flags:
            f.raise_if_set("group reduce")

    def nvlink_bytes_per_gpu(self) -> int:
        """Algorithmic cross-GPU bytes per step per GPU (in + out)."""
        S = self.n * self.es
        if self.variant == "rank_tree2":
            return 2 * (self.G - 1) * S // self.G
        return (self.G - 1) * self.E * S // (self.G * self.G) + (self.G - 1) * S // self.G
