"""One process per GPU: the EST-sharded data-parallel step over torch.distributed.

The ESTs are independent until the one exchange step of a mini-batch, so the
path shards by EST: rank g owns the contiguous rank block
`est_block(g, G, E)` (the reference's assign_ranks, engine.py:169-199).  Per
mini-batch each rank

  1. runs the step kernel in grads-only mode for its ESTs (bt_mlp_step,
     fuse_reduce = 0): forward/backward, loss, TrackedStat, RNG advance;
  2. exchanges the EST gradient slots with one all-gather -- a bit copy, so
     the result is deterministic on any backend (NCCL over NVLink here);
  3. applies the same fixed-order reduce + /E + momentum SGD kernel
     (bt_reduce_update) to all E slots in ascending-rank order with the
     bucket-map rotation, so every rank ends with bitwise-identical weights
     and no parameter broadcast is needed.

No collective ever adds floating-point numbers: NCCL ring/tree allreduce
order depends on the world size, which is exactly what the reference's
determinism levels forbid (§3.3).
"""

from __future__ import annotations

import ctypes as C

import torch
import torch.distributed as dist

from . import _native
from .buckets import build_buckets_initial, rotation_table
from .device import Flags, require_cuda, stream, u64_to_i64
from .errors import ConfigError, NumericError
from .model import PARAM_COUNT, ToyModel
from .prng import TAG_DROPOUT, derive_stream
from .reduction import fanin_code
from .sampling import DataPipeline


def est_block(rank: int, world: int, E: int) -> tuple[int, int]:
    """(first EST, count) of a rank: contiguous, balanced, larger shares first (engine.py:189-193)."""
    if world < 1 or world > E:
        raise ConfigError(f"{world} ranks for only {E} ESTs")
    base, extra = divmod(E, world)
    counts = [base + (1 if i < extra else 0) for i in range(world)]
    return sum(counts[:rank]), counts[rank]


class SlotExchange:
    """All-gather of per-rank EST slot blocks into rank order (a bit copy)."""

    def __init__(self, E: int, width: int, group=None):
        self.group = group
        self.world = dist.get_world_size(group)
        self.rank = dist.get_rank(group)
        self.E, self.width = E, width
        self.blocks = [est_block(r, self.world, E) for r in range(self.world)]
        self.equal = len({c for _, c in self.blocks}) == 1

    def allgather(self, local: torch.Tensor, out: torch.Tensor | None = None) -> torch.Tensor:
        """local: [count_r, width] -> [E, width] with rank r's block at rows [base_r, base_r+count_r)."""
        if out is None:
            out = torch.empty((self.E, self.width), dtype=local.dtype, device=local.device)
        if self.equal and local.is_cuda:
            dist.all_gather_into_tensor(out, local.contiguous(), group=self.group)
            return out
        cmax = max(c for _, c in self.blocks)
        pad = torch.zeros((cmax, self.width), dtype=local.dtype, device=local.device)
        pad[: local.shape[0]] = local
        parts = [torch.empty_like(pad) for _ in range(self.world)]
        dist.all_gather(parts, pad, group=self.group)
        for (base, count), part in zip(self.blocks, parts):
            out[base: base + count] = part[:count]
        return out


class DistributedTrainer:
    """C2-style job sharded over the ranks of the default process group (one GPU each)."""

    def __init__(self, seed=42, max_workers=8, micro_batch=4, dataset_size=1024, lr=0.02, momentum=0.9,
                 dropout_rate=0.5, jitter=0.1, bucket_capacity=64, fanin=2, comm_fanin=2, group=None,
                 exchange: str | None = None):
        """exchange (None: "xdev" where its shape applies, else "allgather"): "xdev" -- the persistent
        lock-step kernel: K mini-batches per launch,
        EST slots stored into every rank's inbox over CUDA IPC peer memory with device-side counters
        (run(K)); "ipc" -- no collective at all: each rank owns a parameter shard and its reduce kernel
        reads every rank's slots and writes every rank's replica through CUDA IPC peer pointers,
        ordered by stream memory operations (paper_2208_14228_b200.peer); "allgather" -- NCCL
        all-gather of the EST slots, then the reduce kernel on every rank."""
        require_cuda()
        self.rank, self.world = dist.get_rank(group), dist.get_world_size(group)
        self.E, self.B = max_workers, micro_batch
        self.base, self.count = est_block(self.rank, self.world, self.E)
        self.lr, self.mu, self.rate, self.jitter, self.seed = lr, momentum, dropout_rate, jitter, seed
        self.comm_fanin = comm_fanin
        self.xchg = SlotExchange(self.E, PARAM_COUNT, group)
        self.params = torch.zeros((2, PARAM_COUNT), dtype=torch.float64, device="cuda")
        self.params[0] = ToyModel.init_random(seed).tensor
        self.stage = torch.empty(PARAM_COUNT, dtype=torch.float64, device="cuda")  # guarded update
        self.fan = torch.full((self.count,), fanin, dtype=torch.int32, device="cuda")
        self.rng = torch.tensor([u64_to_i64(derive_stream(TAG_DROPOUT, seed, self.base + k))
                                 for k in range(self.count)], dtype=torch.int64, device="cuda")
        self.stat_mean = torch.zeros(self.count, dtype=torch.float64, device="cuda")
        self.stat_count = torch.zeros(self.count, dtype=torch.int64, device="cuda")
        self.grads_loc = torch.zeros((self.count, PARAM_COUNT), dtype=torch.float64, device="cuda")
        self.grads_all = torch.zeros((self.E, PARAM_COUNT), dtype=torch.float64, device="cuda")
        self.losses = torch.zeros(self.count, dtype=torch.float64, device="cuda")
        bm = build_buckets_initial(PARAM_COUNT, bucket_capacity)
        self.rot = torch.from_numpy(rotation_table(bm, self.E)).to("cuda") if comm_fanin else None
        self.pipe = DataPipeline(seed, dataset_size, self.E, micro_batch, jitter, 2, 2)
        self.flags = Flags()
        self.step_idx = 0
        if exchange is None:  # the lock-step kernel wherever its shape applies
            exchange = "xdev" if (self.world in (2, 4, 8) and self.E in (4, 8, 16) and self.E % self.world == 0
                                  and micro_batch == 4 and fanin == comm_fanin and fanin in (0, 2)) else "allgather"
        self.exchange = exchange
        self.peer = None
        if exchange == "ipc":
            from .hier import RankBuffers
            from .peer import PeerGroupReducer

            if comm_fanin not in (0, 2):
                raise ConfigError("the IPC reducer supports Sequential and Tree(2) allreduce variants")
            if self.E % self.world:
                raise ConfigError("the IPC reducer needs equal EST blocks per rank")
            self.peer = PeerGroupReducer(
                RankBuffers(self.grads_loc, self.params[0], self.params[1], torch.cuda.current_stream()), self.E,
                "sequential" if comm_fanin == 0 else "tree2_rotated", self.rot, lr, momentum, group)
        elif exchange == "xdev":
            self._init_xdev(group, fanin)
        elif exchange != "allgather":
            raise ConfigError(f"unknown exchange {exchange!r}")

    # ------------------------------------------------------------------ lock-step (xdev)
    KMAX = 128

    def _init_xdev(self, group, fanin: int) -> None:
        """The persistent multi-GPU step: every rank runs K mini-batches in ONE launch of the fused
        step kernel (bt_mlp.cu, n_dev = world), storing its EST slots into every other rank's inbox
        (CUDA IPC peer memory over NVLink) as tagged 8-byte words each mini-batch, polled by the
        receiver; each rank folds all E slots in the canonical order itself.  No host, NCCL or stream operation
        per mini-batch."""
        from .peer import _export, _Opened

        if not (self.E in (4, 8, 16) and self.world in (2, 4, 8) and self.E % self.world == 0 and self.B == 4
                and fanin == self.comm_fanin and fanin in (0, 2)):
            raise ConfigError("the lock-step exchange needs E in {4,8,16} over 2/4/8 ranks, micro-batch 4 and "
                              "one Sequential/Tree(2) variant")
        from .placement import inbox_words

        self.inbox = torch.zeros(inbox_words(self.E), dtype=torch.int64, device="cuda")
        self.xlosses = torch.zeros((self.KMAX, self.E), dtype=torch.float64, device="cuda")
        table = [None] * self.world
        dist.all_gather_object(table, _export(self.inbox), group=group)
        self.opened = _Opened()
        self.xin = [self.inbox.data_ptr() if q == self.rank else self.opened.ptr(*table[q]) for q in range(self.world)]
        torch.cuda.synchronize()
        dist.barrier(group=group)  # every rank's inbox is zero before any launch writes into it

    def xdev_args(self, K: int) -> _native.MlpArgs:
        """The launch of the next K mini-batches (caller keeps the lists tensor alive)."""
        spe = self.pipe.steps_per_epoch
        gs = self.step_idx
        lists, lbase = self.pipe.device_lists(gs // spe, (gs + K - 1) // spe)
        self._xlists = lists
        a = _native.MlpArgs()
        a.E, a.est_base, a.E_total, a.B, a.X, a.K = self.count, self.base, self.E, self.B, 1, K
        a.fuse_reduce, a.est_per_cta = 1, 1
        a.comm_fanin, a.est_fanin_uniform, a.rank_override = self.comm_fanin, self.comm_fanin + 1, -1
        a.rate, a.lr, a.mu, a.jitter = self.rate, self.lr, self.mu, self.jitter
        a.replicas, a.est_fanin, a.rng = self.params.data_ptr(), self.fan.data_ptr(), self.rng.data_ptr()
        a.stat_mean, a.stat_count = self.stat_mean.data_ptr(), self.stat_count.data_ptr()
        a.grads, a.losses = self.grads_loc.data_ptr(), self.xlosses.data_ptr()
        a.rot = self.rot.data_ptr() if self.rot is not None else None
        a.dataset, a.lists, a.dataset_rows = self.pipe.dataset_device.data_ptr(), lists.data_ptr(), self.pipe.dataset_size
        a.seed, a.step0, a.spe, a.epoch_base = self.seed & (2**64 - 1), gs, spe, lbase
        a.flags, a.bar = self.flags.t.data_ptr(), None
        a.n_dev, a.dev_index = self.world, self.rank
        for q in range(self.world):
            a.xin[q] = self.xin[q]
        return a

    def run(self, K: int) -> torch.Tensor:
        """K mini-batches in one lock-step launch (every rank must call run(K) with the same K);
        returns the losses [K][E] (this rank's EST columns filled), on the device."""
        if self.exchange != "xdev":
            raise ConfigError("run(K) is the lock-step exchange's entry point")
        if K < 1 or K > self.KMAX:
            raise ConfigError(f"K must be in [1, {self.KMAX}]")
        a = self.xdev_args(K)
        _native.check(_native.lib().bt_mlp_step(C.byref(a), stream()), "lock-step step")
        self.step_idx += K
        return self.xlosses[:K]

    def step(self) -> torch.Tensor:
        """One mini-batch; returns this rank's per-EST losses (device tensor)."""
        if self.exchange == "xdev":
            return self.run(1)[0, self.base:self.base + self.count]
        spe = self.pipe.steps_per_epoch
        epoch, local = divmod(self.step_idx, spe)
        lists, lbase = self.pipe.device_lists(epoch, epoch)
        a = _native.MlpArgs()
        a.E, a.est_base, a.E_total, a.B, a.X, a.K = self.count, self.base, self.E, self.B, 1, 1
        a.fuse_reduce = 0
        a.est_per_cta = _native.lib().bt_mlp_pick_est_per_cta(self.count, self.B)
        a.comm_fanin, a.rank_override = self.comm_fanin, -1
        a.rate, a.lr, a.mu, a.jitter = self.rate, self.lr, self.mu, self.jitter
        a.replicas, a.est_fanin, a.rng = self.params.data_ptr(), self.fan.data_ptr(), self.rng.data_ptr()
        a.stat_mean, a.stat_count = self.stat_mean.data_ptr(), self.stat_count.data_ptr()
        a.grads, a.losses = self.grads_loc.data_ptr(), self.losses.data_ptr()
        a.dataset, a.lists, a.dataset_rows = self.pipe.dataset_device.data_ptr(), lists.data_ptr(), self.pipe.dataset_size
        a.seed, a.step0, a.spe, a.epoch_base = self.seed & (2**64 - 1), self.step_idx, spe, lbase
        a.flags = self.flags.t.data_ptr()
        _native.check(_native.lib().bt_mlp_step(C.byref(a), stream()), "forward_backward")
        if self.peer is not None:  # fused reduce-scatter + SGD + all-gather over peer memory
            self.peer.step()
            self.step_idx += 1
            return self.losses
        self.xchg.allgather(self.grads_loc, self.grads_all)
        r = _native.ReduceArgs()
        r.dtype, r.mode, r.E, r.fanin, r.n = _native.DTYPE_F64, _native.REDUCE_UPDATE, self.E, self.comm_fanin, PARAM_COUNT
        r.grads[0], r.grads_ld = self.grads_all.data_ptr(), PARAM_COUNT
        r.rot = self.rot.data_ptr() if self.rot is not None else None
        r.param, r.vel = self.params[0].data_ptr(), self.params[1].data_ptr()
        r.param_out, r.vel_out = r.param, r.vel  # in place, guarded: nothing changes on a non-finite step
        r.stage = self.stage.data_ptr()
        r.lr, r.mu, r.flags = self.lr, self.mu, self.flags.t.data_ptr()
        _native.check(_native.lib().bt_reduce_update(C.byref(r), stream()), "reduce_update")
        self.step_idx += 1
        return self.losses

    def close(self) -> None:
        torch.cuda.synchronize()
        if self.peer is not None:
            self.peer.close()
        if getattr(self, "opened", None) is not None:
            self.opened.close()

    def check(self) -> None:
        if self.peer is not None:
            self.peer.check()
        st, detail, _ = self.flags.status()
        if st == 5:
            raise NumericError(f"non-finite synchronized gradient at parameter {detail}")
        if st:
            self.flags.raise_if_set("distributed step")


__all__ = ["est_block", "SlotExchange", "DistributedTrainer", "fanin_code"]
