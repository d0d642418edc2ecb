"""Time-sliced elastic training runtime on the B200 (reference engine.py:1-395).

A job has `max_workers` ESTs with fixed virtual ranks.  Executors host
contiguous rank blocks (`assign_ranks`).  All per-EST state lives in HBM
slots indexed by rank (dropout RNG, TrackedStat, gradient slot), so a
"context switch" is an index change and a layout change never moves it.
The executor replicas are [X][2][161] binary64 blocks.

`run_minibatch` launches ONE fused kernel (bt_mlp.cu) that performs, in the
reference's order: data gather + jitter -> replica agreement -> every EST's
forward/backward -> fixed-order allreduce in executor 0's variant -> /E ->
momentum SGD -> mirror to every replica.  `run_steps` runs K mini-batches in
one persistent launch.  If `engine.allreduce` is replaced (e.g. a test spy,
reference test_engine.py:175-199), the step falls back to the unfused device
path that calls it through this module's global, exactly like the reference.
"""

from __future__ import annotations

import ctypes as C
import struct
from dataclasses import dataclass, field

import numpy as np
import torch

from . import _native
from . import buckets as _buckets
from . import placement
from .buckets import (BucketMap, build_buckets_initial, layout_arrival_perm, rebuild_buckets_first_minibatch,
                      rotation_table)
from .device import DeviceVector, Flags, i64_to_u64, ptr, require_cuda, stream, u64_to_i64
from .errors import ConfigError, CorruptionError, NumericError, StateError
from .model import PARAM_COUNT, Batch, OptState, ToyModel, TrackedStat, rows_tensor, sgd_step
from .prng import TAG_DROPOUT, derive_stream
from .reduction import KernelProfile, fanin_code
from .sampling import DataPipeline

allreduce = _buckets.allreduce  # called through this module global (spy-able, engine.py:310)
_DEVICE_ALLREDUCE = _buckets.allreduce
P = PARAM_COUNT


@dataclass(frozen=True)
class DeterminismMode:
    """d0 fixed-parallelism, d1 elasticity (implies d0), d2 heterogeneity (engine.py:44-80)."""

    d0: bool = True
    d1: bool = False
    d2: bool = False

    def __post_init__(self):
        if self.d1 and not self.d0:
            raise ConfigError("d1 requires d0")

    @classmethod
    def from_label(cls, label: str) -> "DeterminismMode":
        table = {"d0": cls(True), "d1": cls(True, True), "d1d2": cls(True, True, True), "d0d2": cls(True, False, True)}
        key = label.strip().lower()
        if key not in table:
            raise ConfigError(f"unknown determinism mode {label!r}")
        return table[key]

    @property
    def label(self) -> str:
        return {(True, True): "d1d2", (True, False): "d1", (False, True): "d0d2", (False, False): "d0"}[(self.d1, self.d2)]


@dataclass(frozen=True)
class ExecutorSpec:
    """One executor of a layout: device kind and optional pinned EST count."""

    device_kind: str
    threads: int | None = None


@dataclass(frozen=True)
class TrainRunConfig:
    """Everything a run depends on besides the layout (engine.py:117-141)."""

    seed: int
    max_workers: int
    micro_batch: int = 4
    dataset_size: int = 1000
    lr: float = 0.02
    momentum: float = 0.9
    dropout_rate: float = 0.5
    jitter: float = 0.1
    bucket_capacity: int = 64
    worker_slots: int = 2
    prefetch_depth: int = 2
    shuffle: bool = True
    determinism: DeterminismMode = DeterminismMode()
    device_fanins: dict = field(default_factory=lambda: {"cpu": 2})

    def kernel_profile(self, device_kind: str) -> KernelProfile:
        if device_kind not in self.device_fanins:
            raise ConfigError(f"unknown device kind {device_kind!r}")
        if self.determinism.d2:
            return KernelProfile.device_agnostic(device_kind)
        return KernelProfile.native(device_kind, self.device_fanins[device_kind])


# ---------------------------------------------------------------- device state
IO_ROWS = 128  # mini-batches of losses a shard's I/O block holds (the prepared launch's KMAX)


class Shard:
    """One GPU's part of a job: the replicas of the executors placed on it and the slots of
    their ESTs (a contiguous rank block).  Slot arrays are [E] on every shard; only the
    entries of the shard's own ESTs are meaningful there."""

    def __init__(self, index: int, ordinal: int, execs: list[int], ests: list[int], E: int):
        self.index, self.ordinal = index, ordinal
        self.execs, self.ests = list(execs), list(ests)
        self.base, self.count = (self.ests[0] if self.ests else 0), len(self.ests)
        with torch.cuda.device(ordinal):
            self.replicas = torch.zeros((len(execs), 2, P), dtype=torch.float64, device="cuda")  # params | vel
            self.est_fanin = torch.zeros(E, dtype=torch.int32, device="cuda")
            self.rng = torch.zeros(E, dtype=torch.int64, device="cuda")         # u64 bit patterns
            self.stat_mean = torch.zeros(E, dtype=torch.float64, device="cuda")
            self.stat_count = torch.zeros(E, dtype=torch.int64, device="cuda")
            self.grads = torch.zeros((2, E, P), dtype=torch.float64, device="cuda")  # step-parity slots
            # I/O block: IO_ROWS x E per-EST losses, then the 4-word status block -- a launch of K
            # mini-batches writes its losses into the last K rows, so one copy brings losses + status
            self.io = torch.zeros(IO_ROWS * E + 2, dtype=torch.float64, device="cuda")
            self.flags = Flags(self.io[IO_ROWS * E:].view(torch.int32))
            self.bar = torch.zeros(1, dtype=torch.int32, device="cuda")
            # the stream of this shard's lock-step launches: shards sharing one GPU (logical devices)
            # must run concurrently, so each has its own
            self.stream = torch.cuda.Stream()
        self.dataset = None  # this GPU's copy of the resident dataset (multi-GPU jobs)
        self.lists = (None, None)  # (source tensor, this GPU's copy) of the epoch lists
        self.rot = (None, None)

    def on(self, t: torch.Tensor | None, cache: str | None = None) -> torch.Tensor | None:
        """`t` on this shard's GPU (cached per source tensor when `cache` names a slot)."""
        if t is None or t.device.index == self.ordinal:
            return t
        if cache is not None:
            src, mine = getattr(self, cache)
            if src is t:
                return mine
        with torch.cuda.device(self.ordinal):
            mine = t.to(torch.device("cuda", self.ordinal))
        if cache is not None:
            setattr(self, cache, (t, mine))
        return mine


class DeviceState:
    """HBM layout of one job over its GPUs: executor x lives on
    shard `exec_shard[x]` (placement.executor_devices: contiguous blocks over the job's GPUs),
    EST k's slots on the shard of the executor that hosts it."""

    def __init__(self, E: int, ranks: list[tuple[str, list[int]]]):
        require_cuda()
        self.E, self.X = E, len(ranks)
        devs = placement.devices()
        plan = placement.executor_devices(self.X, devs)
        self.shards: list[Shard] = []
        self.exec_loc: list[tuple[Shard, int]] = [None] * self.X
        self.est_owner: list[Shard] = [None] * E
        for i in range(max(plan) + 1):
            execs = [x for x in range(self.X) if plan[x] == i]
            ests = [k for x in execs for k in ranks[x][1]]
            sh = Shard(i, devs[i], execs, ests, E)
            self.shards.append(sh)
            for j, x in enumerate(execs):
                self.exec_loc[x] = (sh, j)
            for k in ests:
                self.est_owner[k] = sh
        if len(self.shards) > 1:
            placement.enable_peer_access([sh.ordinal for sh in self.shards])
        self._snap = None
        self.rot = None
        self.rot_key = None
        self.xstep = None  # the prepared multi-GPU launch (_XdevStep)

    # -- the single-GPU view (one shard: every executor and EST on one device) --------------
    @property
    def multi(self) -> bool:
        return len(self.shards) > 1

    def _one(self) -> Shard:
        if self.multi:
            raise RuntimeError("this job spans several GPUs: address its shards")
        return self.shards[0]

    replicas = property(lambda self: self._one().replicas)
    est_fanin = property(lambda self: self._one().est_fanin)
    rng = property(lambda self: self._one().rng)
    stat_mean = property(lambda self: self._one().stat_mean)
    stat_count = property(lambda self: self._one().stat_count)
    grads = property(lambda self: self._one().grads)
    flags = property(lambda self: self.shards[0].flags)
    bar = property(lambda self: self._one().bar)

    # -- shard-aware access --------------------------------------------------------------------
    def replica(self, x: int) -> torch.Tensor:
        sh, j = self.exec_loc[x]
        return sh.replicas[j]

    def owner(self, k: int) -> Shard:
        return self.est_owner[k]

    def invalidate(self) -> None:
        self._snap = None

    def snapshot(self):
        if self._snap is None:
            rng, mean, cnt = [0] * self.E, [0.0] * self.E, [0] * self.E
            for sh in self.shards:
                r, m, c = sh.rng.tolist(), sh.stat_mean.tolist(), sh.stat_count.tolist()
                for k in sh.ests:
                    rng[k], mean[k], cnt[k] = r[k], m[k], c[k]
            self._snap = (rng, mean, cnt)
        return self._snap

    def load_contexts(self, rng: list[int], mean: list[float], count: list[int]) -> None:
        for sh in self.shards:
            sh.rng.copy_(torch.tensor(rng, dtype=torch.int64))
            sh.stat_mean.copy_(torch.tensor(mean, dtype=torch.float64))
            sh.stat_count.copy_(torch.tensor(count, dtype=torch.int64))
        self.invalidate()

    def load_replicas(self, block: torch.Tensor) -> None:
        """Every executor's replica <- block [2][P]."""
        for sh in self.shards:
            sh.replicas.copy_(block.to(sh.replicas.device).unsqueeze(0).expand_as(sh.replicas))

    def set_fanin(self, fan: np.ndarray) -> None:
        t = torch.from_numpy(fan)
        for sh in self.shards:
            sh.est_fanin.copy_(t)

    def replica_ptrs(self) -> list[int]:
        return [self.replica(x).data_ptr() for x in range(self.X)]


class WorkerContext:
    """All state owned by one EST (engine.py:95-103).

    Detached (host fields) until attached to a DeviceState slot; attached
    contexts read and write their HBM slot."""

    def __init__(self, virtual_rank: int, dropout_rng: int = 0, stat: TrackedStat = TrackedStat(),
                 pending_grads=None, minibatch_idx: int = 0):
        self.virtual_rank = virtual_rank
        self._rng = dropout_rng
        self._stat = stat
        self.pending_grads = pending_grads
        self.minibatch_idx = minibatch_idx
        self._dev: DeviceState | None = None

    def attach(self, dev: DeviceState) -> None:
        k = self.virtual_rank
        sh = dev.owner(k)
        sh.rng[k] = u64_to_i64(self._rng)
        sh.stat_mean[k] = self._stat.running_mean
        sh.stat_count[k] = self._stat.update_count
        dev.invalidate()
        self._dev = dev

    @property
    def dropout_rng(self) -> int:
        if self._dev is None:
            return self._rng
        return i64_to_u64(self._dev.snapshot()[0][self.virtual_rank])

    @dropout_rng.setter
    def dropout_rng(self, v: int) -> None:
        if self._dev is None:
            self._rng = v
        else:
            self._dev.owner(self.virtual_rank).rng[self.virtual_rank] = u64_to_i64(v)
            self._dev.invalidate()

    @property
    def stat(self) -> TrackedStat:
        if self._dev is None:
            return self._stat
        _, means, counts = self._dev.snapshot()
        return TrackedStat(means[self.virtual_rank], int(counts[self.virtual_rank]))

    @stat.setter
    def stat(self, s: TrackedStat) -> None:
        if self._dev is None:
            self._stat = s
        else:
            sh = self._dev.owner(self.virtual_rank)
            sh.stat_mean[self.virtual_rank] = s.running_mean
            sh.stat_count[self.virtual_rank] = s.update_count
            self._dev.invalidate()

    def _key(self):
        pg = None if self.pending_grads is None else list(self.pending_grads)
        return (self.virtual_rank, self.dropout_rng, self.stat, pg, self.minibatch_idx)

    def __eq__(self, other) -> bool:
        return isinstance(other, WorkerContext) and self._key() == other._key()

    __hash__ = None

    def __repr__(self) -> str:
        return (f"WorkerContext(virtual_rank={self.virtual_rank}, dropout_rng={self.dropout_rng:#x}, "
                f"stat={self.stat}, minibatch_idx={self.minibatch_idx})")


class ExecutorState:
    """A device context hosting a replica shared by its ESTs (engine.py:106-114).

    `model`/`opt` are views of this executor's block of DeviceState.replicas."""

    def __init__(self, device_kind: str, kernel_profile: KernelProfile, assigned: list[int], dev: DeviceState,
                 index: int, lr: float, momentum: float):
        self.device_kind = device_kind
        self.kernel_profile = kernel_profile
        self.assigned = assigned
        self._dev, self._x = dev, index
        self._lr, self._mu = lr, momentum

    @property
    def device(self) -> torch.device:
        """The GPU this executor runs on (placement.executor_devices)."""
        return self._dev.replica(self._x).device

    @property
    def model(self) -> ToyModel:
        return ToyModel(self._dev.replica(self._x)[0])

    @model.setter
    def model(self, m: ToyModel) -> None:
        self._dev.replica(self._x)[0].copy_(m.tensor)

    @property
    def opt(self) -> OptState:
        return OptState(self._lr, self._mu, self._dev.replica(self._x)[1])

    @opt.setter
    def opt(self, o: OptState) -> None:
        self._lr, self._mu = o.lr, o.momentum
        self._dev.replica(self._x)[1].copy_(o.tensor)


@dataclass
class TrainingState:
    """The unit of checkpointing (engine.py:144-162) plus its device slots."""

    cfg: TrainRunConfig
    contexts: list
    executors: list
    bucket_map: BucketMap
    pipeline: DataPipeline
    global_step: int = 0
    epoch: int = 0
    rebuild_pending: bool = False
    dev: DeviceState | None = None
    _fast: object = field(default=None, repr=False, compare=False)  # prepared launch (_FastStep)

    @property
    def max_workers(self) -> int:
        return self.cfg.max_workers

    def layout_key(self) -> list[tuple[str, int]]:
        return [(ex.device_kind, len(ex.assigned)) for ex in self.executors]


def floats_to_bytes(values) -> bytes:
    if isinstance(values, DeviceVector):
        return values.to_bytes()
    return struct.pack(f"<{len(values)}d", *values)


def assign_ranks(specs: list[ExecutorSpec], max_workers: int) -> list[tuple[str, list[int]]]:
    """Contiguous rank blocks (engine.py:169-199): pinned counts must sum to
    max_workers; otherwise balanced, larger shares first."""
    if not specs:
        raise ConfigError("layout needs at least one executor")
    pinned = [s.threads for s in specs]
    if any(t is not None for t in pinned):
        if any(t is None for t in pinned):
            raise ConfigError("either all executors or none may pin thread counts")
        if any(t < 1 for t in pinned):
            raise ConfigError("executor thread counts must be >= 1")
        if sum(pinned) != max_workers:
            raise ConfigError(f"thread counts sum to {sum(pinned)}, expected {max_workers}")
        counts = list(pinned)
    else:
        if len(specs) > max_workers:
            raise ConfigError(f"{len(specs)} executors for only {max_workers} workers")
        base, extra = divmod(max_workers, len(specs))
        counts = [base + (i < extra) for i in range(len(specs))]
    out, start = [], 0
    for spec, c in zip(specs, counts):
        out.append((spec.device_kind, list(range(start, start + c))))
        start += c
    return out


def _build_executors(cfg: TrainRunConfig, layout, dev: DeviceState, lr: float, mu: float) -> list[ExecutorState]:
    execs = []
    fan = np.zeros(cfg.max_workers, dtype=np.int32)
    for x, (kind, ranks) in enumerate(assign_ranks(list(layout), cfg.max_workers)):
        prof = cfg.kernel_profile(kind)
        f = fanin_code(prof.reduce_variant)
        fan[ranks] = f
        execs.append(ExecutorState(kind, prof, ranks, dev, x, lr, mu))
    dev.set_fanin(fan)
    return execs


def _new_pipeline(cfg: TrainRunConfig, dataset_dev=None) -> DataPipeline:
    pipe = DataPipeline(cfg.seed, cfg.dataset_size, cfg.max_workers, cfg.micro_batch, cfg.jitter, cfg.worker_slots,
                        cfg.prefetch_depth, cfg.shuffle)
    if dataset_dev is not None:
        pipe._dataset_dev = dataset_dev
    return pipe


def init_training(cfg: TrainRunConfig, layout: list[ExecutorSpec]) -> TrainingState:
    """Fresh state on the layout (engine.py:202-243), built in HBM."""
    for spec in layout:
        cfg.kernel_profile(spec.device_kind)  # ConfigError on unknown kinds before allocating
    ranks = assign_ranks(list(layout), cfg.max_workers)
    dev = DeviceState(cfg.max_workers, ranks)
    init = ToyModel.init_random(cfg.seed)
    dev.load_replicas(torch.stack([init.tensor, torch.zeros_like(init.tensor)]))
    executors = _build_executors(cfg, layout, dev, cfg.lr, cfg.momentum)
    contexts = []
    for k in range(cfg.max_workers):
        ctx = WorkerContext(k, derive_stream(TAG_DROPOUT, cfg.seed, k), TrackedStat())
        contexts.append(ctx)
    dev.load_contexts([u64_to_i64(c._rng) for c in contexts], [0.0] * cfg.max_workers, [0] * cfg.max_workers)
    for c in contexts:
        c._dev = dev
    return TrainingState(cfg, contexts, executors, build_buckets_initial(P, cfg.bucket_capacity),
                         _new_pipeline(cfg), rebuild_pending=not cfg.determinism.d1, dev=dev)


def check_replica_agreement(ts: TrainingState) -> None:
    """Every executor's params+velocity must be bitwise equal (engine.py:246-258), on the device:
    one compare kernel on the first GPU reads every replica (peer loads from the other GPUs)."""
    dev = ts.dev
    if dev.X < 2:
        return
    ptrs = (C.c_void_p * dev.X)(*dev.replica_ptrs())
    sh0 = dev.shards[0]
    with torch.cuda.device(sh0.ordinal):
        _native.check(_native.lib().bt_replica_check(ptrs, dev.X, 2 * P * 8, ptr(sh0.flags.t), stream()),
                      "check_replica_agreement")
    st, detail, _ = dev.flags.status()
    if st:
        dev.flags.reset()
        if st == 6:
            kind = ts.executors[detail].device_kind if 0 <= detail < len(ts.executors) else "?"
            raise CorruptionError(f"model/optimizer replica on executor of kind {kind!r} diverged")
        raise RuntimeError(f"replica check failed with status {st}")


def split_by_rank(global_batch: Batch, max_workers: int) -> list[Batch]:
    """Row t belongs to rank t mod P (engine.py:261-268)."""
    if len(global_batch) == 0 or len(global_batch) % max_workers != 0:
        raise ConfigError(f"global batch of {len(global_batch)} rows is not divisible by {max_workers}")
    return [global_batch[k::max_workers] for k in range(max_workers)]


def _comm_variant(ts: TrainingState):
    return ts.executors[0].kernel_profile.reduce_variant  # engine.py:309


def _rot_tensor(ts: TrainingState):
    variant = _comm_variant(ts)
    if fanin_code(variant) == 0:
        return None
    dev = ts.dev
    rk = dev.rot_key
    if rk is not None and rk[0] is ts.bucket_map and rk[1] == ts.cfg.max_workers:  # the per-call case
        return dev.rot
    key = (ts.bucket_map, ts.cfg.max_workers)
    if rk != key:
        with torch.cuda.device(dev.shards[0].ordinal):
            dev.rot = torch.from_numpy(rotation_table(ts.bucket_map, ts.cfg.max_workers)).to("cuda")
        dev.rot_key = key
    return dev.rot


def _step_args(ts: TrainingState, K: int, B: int, rows: torch.Tensor | None, losses: torch.Tensor,
               trace: torch.Tensor | None, fuse: bool = True) -> tuple[_native.MlpArgs, list]:
    cfg, dev = ts.cfg, ts.dev
    ex0 = ts.executors[0]
    keep = []
    a = _native.MlpArgs()
    a.E = a.E_total = cfg.max_workers
    a.est_base = 0
    a.B, a.X, a.K = B, dev.X, K
    a.fuse_reduce = int(fuse)
    a.est_per_cta = _native.lib().bt_mlp_pick_est_per_cta(cfg.max_workers, B)
    a.comm_fanin = fanin_code(_comm_variant(ts))
    fans = {fanin_code(ex.kernel_profile.reduce_variant) for ex in ts.executors}
    a.est_fanin_uniform = fans.pop() + 1 if len(fans) == 1 else 0  # lets the launcher specialise
    a.rank_override = -1
    a.rate, a.lr, a.mu, a.jitter = float(cfg.dropout_rate), float(ex0._lr), float(ex0._mu), float(cfg.jitter)
    a.replicas, a.est_fanin, a.rng = ptr(dev.replicas), ptr(dev.est_fanin), ptr(dev.rng)
    a.stat_mean, a.stat_count, a.grads, a.losses = ptr(dev.stat_mean), ptr(dev.stat_count), ptr(dev.grads), ptr(losses)
    rot = _rot_tensor(ts) if fuse else None
    a.rot = ptr(rot)
    a.seed = cfg.seed & (2**64 - 1)
    a.step0 = ts.global_step
    a.spe = ts.pipeline.steps_per_epoch
    if rows is not None:
        a.rows = ptr(rows)
    else:
        first = ts.global_step // a.spe
        last = (ts.global_step + K - 1) // a.spe
        lists, base = ts.pipeline.device_lists(first, last)
        keep.append(lists)
        a.dataset, a.lists, a.epoch_base = ptr(ts.pipeline.dataset_device), ptr(lists), base
        a.dataset_rows = cfg.dataset_size
    a.flags, a.bar, a.param_trace = ptr(dev.flags.t), ptr(dev.bar), ptr(trace)
    keep += [rot, rows, losses, trace]
    return a, keep


_FITS: dict = {}


def _fused_fits(cfg, B: int | None = None) -> bool:
    """Whether one fused launch holds the whole step on chip (bt_mlp_fused_fits); a pure function of
    (E, B), cached (it is asked on every run_minibatch / run_steps call)."""
    key = (cfg.max_workers, cfg.micro_batch if B is None else B)
    hit = _FITS.get(key)
    if hit is not None:
        return hit
    a = _native.MlpArgs()
    a.E = a.E_total = cfg.max_workers
    a.B = cfg.micro_batch if B is None else B
    a.K, a.fuse_reduce = 1, 1
    a.est_per_cta = _native.lib().bt_mlp_pick_est_per_cta(a.E, a.B)
    _FITS[key] = ok = bool(_native.lib().bt_mlp_fused_fits(C.byref(a)))
    return ok


def _raise_step_error(ts: TrainingState, st: int, detail: int, what: str) -> None:
    for sh in ts.dev.shards:
        sh.flags.reset()
    if st == 6:
        raise CorruptionError(f"{what}: an executor's model/optimizer replica diverged")
    if st == 5:
        raise NumericError(f"{what}: non-finite synchronized gradient")
    raise RuntimeError(f"{what}: device failure status {st}: {_native.last_error()}")


def _finish_steps(ts: TrainingState, nsteps: int) -> None:
    for ctx in ts.contexts:
        ctx.pending_grads = None
        ctx.minibatch_idx += nsteps
    ts.global_step += nsteps
    ts.epoch = ts.global_step // ts.pipeline.steps_per_epoch
    if nsteps and ts.rebuild_pending:
        # d0: after the first post-boot mini-batch the bucket map is rebuilt
        # from the layout-keyed arrival order (engine.py:323-328).
        perm = layout_arrival_perm(P, ts.layout_key())
        ts.bucket_map = rebuild_buckets_first_minibatch(perm, ts.cfg.bucket_capacity)
        ts.rebuild_pending = False


def _raw_stream() -> int:
    return torch._C._cuda_getCurrentRawStream(torch.cuda.current_device())


class _FastStep:
    """The sampler-mode launch of run_minibatch / run_steps, prepared once per TrainingState:
    the argument block with its fixed pointers, and pinned host buffers that bt_mlp_run fills
    with the per-EST losses and the status words (one C-ABI call and one sync per call)."""

    KMAX = IO_ROWS

    def __init__(self, ts: TrainingState):
        cfg = ts.cfg
        self.E = cfg.max_workers
        self.fits = _fused_fits(cfg)
        # the shard's I/O block: a K-mini-batch launch writes its losses into the last K rows, which the
        # status words follow -- so bt_mlp_run brings both back in one copy into the same layout on the host
        io = ts.dev.shards[0].io
        self.io_ptr = io.data_ptr()
        self.host_io = torch.zeros(io.numel(), dtype=torch.float64).pin_memory()
        self.host_io_ptr = self.host_io.data_ptr()
        io_np = self.host_io.numpy()
        self.rows_np = io_np[:self.KMAX * self.E].reshape(self.KMAX, self.E)
        self.status_np = io_np[self.KMAX * self.E:].view(np.int32)
        self.losses_np = self.rows_np
        self.a, self.keep = _step_args(ts, 1, cfg.micro_batch, None, io, None) if self.fits else (None, [])
        self.dev = ts.dev
        # per-call host work is part of every run_minibatch: the argument block's reference, the entry points
        # and the device ordinal are looked up once, and fields that rarely change are written only on change
        self.aref = C.byref(self.a) if self.fits else None
        lib = _native.lib()
        self.run_fn, self.run_sampled_fn = lib.bt_mlp_run, lib.bt_mlp_run_sampled
        self.ordinal = ts.dev.shards[0].ordinal
        self._set = None  # (rot tensor, lr, mu) last written into the argument block

    def run(self, ts: TrainingState, K: int) -> int:
        """Launch K mini-batches from ts.global_step; returns the device status word."""
        a = self.a
        gs = ts.global_step
        pipe = ts.pipeline
        spe = pipe.steps_per_epoch
        e0, e1 = gs // spe, (gs + K - 1) // spe
        rot = _rot_tensor(ts)
        ex0 = ts.executors[0]
        a.K, a.step0 = K, gs
        key = (rot, ex0._lr, ex0._mu)
        if self._set is None or key[0] is not self._set[0] or key[1:] != self._set[1:]:
            a.rot = ptr(rot)
            a.lr, a.mu = float(ex0._lr), float(ex0._mu)
            self._set = key
        off = 8 * (self.KMAX - K) * self.E  # the launch's losses end where the status words begin
        a.losses = self.io_ptr + off
        lh = self.host_io_ptr + off
        sp = torch._C._cuda_getCurrentRawStream(self.ordinal)
        if pipe.lists_resident(e0, e1):
            lists, base = pipe._lists_dev, pipe._lists_dev_base
            self.keep = lists
            a.lists, a.epoch_base = lists.data_ptr(), base
            st = self.run_fn(self.aref, lh, None, sp)
        else:  # the epochs' lists are made on the host inside the native call, copied, then the launch
            count = max(e1 - e0 + 1, pipe.EPOCH_WINDOW)
            stage, lists = pipe.reserve_lists(e0, count)
            self.keep = lists
            st = self.run_sampled_fn(self.aref, pipe.seed & (2**64 - 1), pipe.dataset_size, int(pipe.shuffle), e0,
                                     count, stage, lists.data_ptr(), lh, None, sp)
            if st:
                pipe.drop_lists()
        if st:
            _native.check(st, "run_minibatch")
        self.losses_np = self.rows_np[self.KMAX - K:]
        self.dev._snap = None  # (DeviceState.invalidate)
        return int(self.status_np[0])


class _XdevStep:
    """The lock-step multi-GPU launch (bt_mlp.cu with n_dev > 1) of a job whose executors span
    several GPUs: every GPU runs the fused step for its EST block, stores its EST gradient slots
    into every other GPU's inbox over NVLink each mini-batch and folds all E slots in the canonical
    rank order itself -- the same bits on every GPU and as on one GPU."""

    KMAX = 128

    @staticmethod
    def eligible(ts: TrainingState) -> bool:
        dev, cfg = ts.dev, ts.cfg
        n = len(dev.shards)
        fans = {fanin_code(ex.kernel_profile.reduce_variant) for ex in ts.executors}
        return (n in (2, 4, 8) and cfg.max_workers in (4, 8, 16) and cfg.micro_batch == 4
                and len({sh.count for sh in dev.shards}) == 1 and cfg.max_workers % n == 0
                and len(fans) == 1 and fans == {fanin_code(_comm_variant(ts))} and fans <= {0, 2})

    def __init__(self, ts: TrainingState):
        dev, cfg = ts.dev, ts.cfg
        E, n = cfg.max_workers, len(dev.shards)
        self.dev, self.n = dev, n
        self.group = placement.XGroup([sh.ordinal for sh in dev.shards], E)
        fan = fanin_code(_comm_variant(ts))
        xin = self.group.table()
        lib = _native.lib()
        self.args, self.keep = [], []
        self.losses_dev, self.host_losses, self.host_status = [], [], []
        ds = ts.pipeline.dataset_device
        for i, sh in enumerate(dev.shards):
            with torch.cuda.device(sh.ordinal):
                losses = torch.zeros((self.KMAX, E), dtype=torch.float64, device="cuda")
            sh.dataset = sh.on(ds) if sh.dataset is None else sh.dataset
            a = _native.MlpArgs()
            a.E, a.est_base, a.E_total, a.B, a.X, a.K = sh.count, sh.base, E, cfg.micro_batch, len(sh.execs), 1
            a.fuse_reduce, a.est_per_cta = 1, 1
            a.comm_fanin, a.est_fanin_uniform, a.rank_override = fan, fan + 1, -1
            a.rate, a.jitter = float(cfg.dropout_rate), float(cfg.jitter)
            a.replicas = sh.replicas.data_ptr()
            a.est_fanin = sh.est_fanin.data_ptr() + 4 * sh.base
            a.rng, a.stat_mean = sh.rng.data_ptr() + 8 * sh.base, sh.stat_mean.data_ptr() + 8 * sh.base
            a.stat_count = sh.stat_count.data_ptr() + 8 * sh.base
            a.grads, a.losses = sh.grads.data_ptr(), losses.data_ptr()
            a.dataset, a.dataset_rows = sh.dataset.data_ptr(), cfg.dataset_size
            a.seed, a.spe = cfg.seed & (2**64 - 1), ts.pipeline.steps_per_epoch
            a.flags, a.bar = sh.flags.t.data_ptr(), sh.bar.data_ptr()
            a.n_dev, a.dev_index = n, i
            for q in range(n):
                a.xin[q] = xin[q]
                a.xrep[q] = dev.shards[q].replicas.data_ptr()  # launch-start agreement of every GPU
            self.args.append(a)
            self.losses_dev.append(losses)
            self.host_losses.append(torch.empty((self.KMAX, E), dtype=torch.float64).pin_memory())
            self.host_status.append(torch.zeros(4, dtype=torch.int32).pin_memory())
        self.status_np = [t.numpy() for t in self.host_status]
        self.losses_np = [t.numpy() for t in self.host_losses]
        P_ = C.POINTER(_native.MlpArgs)
        self._argv = (P_ * n)(*[C.pointer(a) for a in self.args])
        self._devs = (C.c_int32 * n)(*[sh.ordinal for sh in dev.shards])
        self._lh = (C.c_void_p * n)(*[t.data_ptr() for t in self.host_losses])
        self._sh = (C.c_void_p * n)(*[t.data_ptr() for t in self.host_status])
        self.lib = lib

    def run(self, ts: TrainingState, K: int, trace: torch.Tensor | None = None) -> tuple[int, int, int, np.ndarray]:
        """K mini-batches from ts.global_step on every GPU; returns (status, detail, failed step,
        losses [K][E]).  trace [K][P] on the first GPU: the parameters after every mini-batch."""
        gs, spe = ts.global_step, ts.pipeline.steps_per_epoch
        lists, base = ts.pipeline.device_lists(gs // spe, (gs + K - 1) // spe)
        rot = _rot_tensor(ts)
        ex0 = ts.executors[0]
        keep = []
        for a, sh in zip(self.args, self.dev.shards):
            ls, rt = sh.on(lists, "lists"), sh.on(rot, "rot")
            keep += [ls, rt]
            a.K, a.step0, a.lists, a.epoch_base = K, gs, ls.data_ptr(), base
            a.rot = ptr(rt)
            a.lr, a.mu = float(ex0._lr), float(ex0._mu)
            a.param_trace = None
        self.args[0].param_trace = ptr(trace)
        for sh in self.dev.shards:  # after everything already queued on the GPU's current stream
            sh.stream.wait_stream(torch.cuda.current_stream(sh.ordinal))
        streams = (C.c_void_p * self.n)(*[sh.stream.cuda_stream for sh in self.dev.shards])
        _native.check(self.lib.bt_mlp_run_group(self._argv, self._devs, streams, self.n, self._lh, self._sh),
                      "run_minibatch (multi-GPU)")
        self.dev.invalidate()
        out = np.empty((K, self.dev.E), dtype=np.float64)
        for sh, l in zip(self.dev.shards, self.losses_np):
            out[:, sh.base:sh.base + sh.count] = l[:K, sh.base:sh.base + sh.count]
        sts = [(int(x[0]), int(x[1]), int(x[2])) for x in self.status_np]
        bad = [t for t in sts if t[0]]
        if not bad:
            return 0, 0, 0, out
        for sh in self.dev.shards:
            sh.flags.reset()
        self.dev.xstep = None  # a retry of the same mini-batch reuses its tags: fresh inboxes next time
        worst = next((t for t in bad if t[0] == 6), None) or next((t for t in bad if t[0] != 9), bad[0])
        return worst[0], worst[1], worst[2], out


def _xdev(ts: TrainingState) -> _XdevStep | None:
    dev = ts.dev
    if not dev.multi or not _XdevStep.eligible(ts):
        return None
    if dev.xstep is None:
        dev.xstep = _XdevStep(ts)
    return dev.xstep


def _grads_multi(ts: TrainingState, B: int, rows) -> tuple[torch.Tensor, list[float]]:
    """Unfused multi-GPU step, part 1: every GPU computes its ESTs' forward/backward (grads-only
    launch of the step kernel); the EST gradient slots are gathered on the first GPU in rank order
    (bit copies).  Returns (grads [E][P] on GPU 0, per-EST losses)."""
    cfg, dev = ts.cfg, ts.dev
    E = cfg.max_workers
    spe = ts.pipeline.steps_per_epoch
    gs = ts.global_step
    lists, lbase = (None, 0) if rows is not None else ts.pipeline.device_lists(gs // spe, gs // spe)
    sh0 = dev.shards[0]
    with torch.cuda.device(sh0.ordinal):
        gall = torch.empty((E, P), dtype=torch.float64, device="cuda")
    losses = [0.0] * E
    for sh in dev.shards:
        with torch.cuda.device(sh.ordinal):
            lt = torch.zeros(max(sh.count, 1), dtype=torch.float64, device="cuda")
            a = _native.MlpArgs()
            a.E, a.est_base, a.E_total, a.B, a.X, a.K = sh.count, sh.base, E, B, len(sh.execs), 1
            a.fuse_reduce = 0
            a.est_per_cta = _native.lib().bt_mlp_pick_est_per_cta(sh.count, B)
            a.comm_fanin, a.rank_override = fanin_code(_comm_variant(ts)), -1
            a.rate, a.jitter = float(cfg.dropout_rate), float(cfg.jitter)
            a.replicas = sh.replicas.data_ptr()
            a.est_fanin = sh.est_fanin.data_ptr() + 4 * sh.base
            a.rng, a.stat_mean = sh.rng.data_ptr() + 8 * sh.base, sh.stat_mean.data_ptr() + 8 * sh.base
            a.stat_count = sh.stat_count.data_ptr() + 8 * sh.base
            a.grads, a.losses = sh.grads.data_ptr() + 8 * sh.base * P, lt.data_ptr()
            a.seed, a.step0, a.spe = cfg.seed & (2**64 - 1), gs, spe
            keep = []
            if rows is not None:
                r = sh.on(rows)
                keep.append(r)
                a.rows = r.data_ptr()
            else:
                if sh.dataset is None:
                    sh.dataset = sh.on(ts.pipeline.dataset_device)
                ls = sh.on(lists, "lists")
                keep.append(ls)
                a.dataset, a.lists, a.epoch_base, a.dataset_rows = sh.dataset.data_ptr(), ls.data_ptr(), lbase, cfg.dataset_size
            a.flags, a.bar = sh.flags.t.data_ptr(), sh.bar.data_ptr()
            _native.check(_native.lib().bt_mlp_step(C.byref(a), stream()), "forward_backward")
            st, detail, _ = sh.flags.status()
            if st:
                _raise_step_error(ts, st, detail, "run_minibatch")
            vals = lt.tolist()
            for j in range(sh.count):
                losses[sh.base + j] = vals[j]
        gall[sh.base:sh.base + sh.count].copy_(sh.grads[0, sh.base:sh.base + sh.count])
    dev.invalidate()
    return gall, losses


def _run_minibatch_multi(ts: TrainingState, B: int, rows) -> list[float]:
    """The same step with its seams exposed across GPUs: per-GPU forward/backward -> the EST slots
    gathered in rank order -> engine.allreduce -> sgd_step -> mirrored to every executor (the
    reference's call sequence, engine.py:288-315; also the path of a spied allreduce)."""
    dev = ts.dev
    check_replica_agreement(ts)
    st, detail, _ = dev.shards[0].flags.status()
    if st:
        _raise_step_error(ts, st, detail, "run_minibatch")
    gall, losses = _grads_multi(ts, B, rows)
    with torch.cuda.device(dev.shards[0].ordinal):
        for ex in ts.executors:
            for rank in ex.assigned[:-1]:  # non-final ESTs park their gradients (engine.py:305-307)
                ts.contexts[rank].pending_grads = DeviceVector(gall[rank].clone())
        synced = globals()["allreduce"]([DeviceVector(gall[r]) for r in range(ts.cfg.max_workers)], ts.bucket_map,
                                        _comm_variant(ts))
        ex0 = ts.executors[0]
        new_model, new_opt = sgd_step(ex0.model, ex0.opt, synced)
        for ex in ts.executors:
            ex.model = new_model
            ex.opt = new_opt
    _finish_steps(ts, 1)
    return losses


def _fast(ts: TrainingState) -> _FastStep:
    fs = ts._fast
    if fs is None or fs.dev is not ts.dev:
        fs = ts._fast = _FastStep(ts)
    return fs


def run_minibatch(ts: TrainingState, global_batch: Batch | None = None) -> list[float]:
    """One mini-batch; returns per-EST losses by ascending rank (engine.py:271-329)."""
    cfg = ts.cfg
    E = cfg.max_workers
    rows = None
    if global_batch is not None:
        split_by_rank(global_batch, E)  # validation (ConfigError)
        B = len(global_batch) // E
        rows = rows_tensor(global_batch)
    else:
        B = cfg.micro_batch
        ts.pipeline.advance_all(ts.global_step)
        if ts.dev.multi:
            xs = _xdev(ts) if globals()["allreduce"] is _DEVICE_ALLREDUCE else None
            if xs is not None:
                st, detail, _, out = xs.run(ts, 1)
                if st:
                    _raise_step_error(ts, st, detail, "run_minibatch")
                _finish_steps(ts, 1)
                return out[0].tolist()
            return _run_minibatch_multi(ts, B, None)
        if globals()["allreduce"] is _DEVICE_ALLREDUCE:
            fs = _fast(ts)
            if fs.fits:
                st = fs.run(ts, 1)
                if st:
                    _raise_step_error(ts, st, int(fs.status_np[1]), "run_minibatch")
                out = fs.losses_np[0].tolist()
                _finish_steps(ts, 1)
                return out
    if ts.dev.multi:  # an explicit global batch over several GPUs
        return _run_minibatch_multi(ts, B, rows)
    if globals()["allreduce"] is not _DEVICE_ALLREDUCE or not _fused_fits(cfg, B):
        # spied allreduce seam, or too many ESTs for on-chip slots: kernels per seam
        return _run_minibatch_unfused(ts, B, rows)
    losses = torch.empty((1, E), dtype=torch.float64, device="cuda")
    a, keep = _step_args(ts, 1, B, rows, losses, None)
    _native.check(_native.lib().bt_mlp_step(C.byref(a), stream()), "run_minibatch")
    st, detail, _ = ts.dev.flags.status()  # one sync per step (the API returns host losses)
    ts.dev.invalidate()
    if st:
        _raise_step_error(ts, st, detail, "run_minibatch")
    out = losses[0].tolist()
    _finish_steps(ts, 1)
    return out


def _run_minibatch_unfused(ts: TrainingState, B: int, rows) -> list[float]:
    """Same step, seams exposed: fwd/bwd kernel -> engine.allreduce -> sgd_step -> mirror."""
    cfg, dev = ts.cfg, ts.dev
    E = cfg.max_workers
    check_replica_agreement(ts)
    losses = torch.empty((1, E), dtype=torch.float64, device="cuda")
    a, keep = _step_args(ts, 1, B, rows, losses, None, fuse=False)
    _native.check(_native.lib().bt_mlp_step(C.byref(a), stream()), "forward_backward")
    st, detail, _ = dev.flags.status()
    dev.invalidate()
    if st:
        _raise_step_error(ts, st, detail, "run_minibatch")
    grads = dev.grads[0]
    for ex in ts.executors:
        for rank in ex.assigned[:-1]:  # non-final ESTs park their gradients (engine.py:305-307)
            ts.contexts[rank].pending_grads = DeviceVector(grads[rank].clone())
    synced = globals()["allreduce"]([DeviceVector(grads[r]) for r in range(E)], ts.bucket_map, _comm_variant(ts))
    ex0 = ts.executors[0]
    new_model, new_opt = sgd_step(ex0.model, ex0.opt, synced)
    for ex in ts.executors:
        ex.model = new_model
        ex.opt = new_opt
    out = losses[0].tolist()
    _finish_steps(ts, 1)
    return out


def run_steps(ts: TrainingState, K: int, trace: bool = False):
    """K mini-batches from the pipeline in one persistent launch.

    Returns (losses [K][E] numpy, params-after-each-step [K][161] numpy or None).
    Identical bits to K calls of run_minibatch."""
    if K < 1:
        raise ConfigError("K must be >= 1")
    if ts.dev.multi:
        return _run_steps_multi(ts, K, trace)
    if ts.rebuild_pending or globals()["allreduce"] is not _DEVICE_ALLREDUCE or not _fused_fits(ts.cfg):
        # one mini-batch at a time: the d0 rebuild after step 0, a spied seam,
        # or a job too large for the fused launch (run_minibatch goes unfused)
        out, tr = [run_minibatch(ts)], ([ts.executors[0].model.values.tolist()] if trace else None)
        while len(out) < K and (ts.rebuild_pending or globals()["allreduce"] is not _DEVICE_ALLREDUCE
                                or not _fused_fits(ts.cfg)):
            out.append(run_minibatch(ts))
            if trace:
                tr.append(ts.executors[0].model.values.tolist())
        if len(out) == K:
            return np.array(out), (np.array(tr) if trace else None)
        rest, rtr = run_steps(ts, K - len(out), trace)
        return np.concatenate([np.array(out), rest]), (np.concatenate([np.array(tr), rtr]) if trace else None)
    cfg = ts.cfg
    E = cfg.max_workers
    gs = ts.global_step
    ts.pipeline.advance_all(gs)  # progress check (ProgressError) before anything runs
    if not trace and K <= _FastStep.KMAX:
        fs = _fast(ts)
        st = fs.run(ts, K)
        failed = int(fs.status_np[2])
        out = fs.losses_np[:K].copy()
    else:
        out, st, failed = None, None, 0
    if st is not None:
        done = K if not st else (failed if st == 5 else 0)
        ts.pipeline.advance_range(gs + 1, min(K, done + (1 if st == 5 else 0)) - 1)
        if st:
            _finish_steps(ts, done)
            _raise_step_error(ts, st, int(fs.status_np[1]), f"run_steps (mini-batch {ts.global_step})")
        _finish_steps(ts, K)
        return out, None
    losses = torch.empty((K, E), dtype=torch.float64, device="cuda")
    tr = torch.empty((K, P), dtype=torch.float64, device="cuda") if trace else None
    a, keep = _step_args(ts, K, cfg.micro_batch, None, losses, tr)
    _native.check(_native.lib().bt_mlp_step(C.byref(a), stream()), "run_steps")
    st, detail, failed = ts.dev.flags.status()
    ts.dev.invalidate()
    done = K if not st else (failed if st == 5 else 0)
    # the failing mini-batch's batches were consumed too (engine.py:282 precedes the sync)
    for s in range(1, min(K, done + (1 if st == 5 else 0))):
        ts.pipeline.advance_all(gs + s)
    if st:
        _finish_steps(ts, done)
        _raise_step_error(ts, st, detail, f"run_steps (mini-batch {ts.global_step})")
    _finish_steps(ts, K)
    return losses.cpu().numpy(), (tr.cpu().numpy() if trace else None)


def _run_steps_multi(ts: TrainingState, K: int, trace: bool):
    """run_steps over several GPUs: one lock-step launch per GPU for up to _XdevStep.KMAX
    mini-batches at a time (or mini-batch by mini-batch on the seam path)."""
    out, tr = [], []
    while len(out) < K:
        xs = None
        if not ts.rebuild_pending and globals()["allreduce"] is _DEVICE_ALLREDUCE:
            xs = _xdev(ts)
        if xs is None:
            out.append(run_minibatch(ts))
            if trace:
                tr.append(ts.executors[0].model.values.tolist())
            continue
        n = min(K - len(out), _XdevStep.KMAX)
        gs = ts.global_step
        ts.pipeline.advance_all(gs)
        tt = None
        if trace:
            with torch.cuda.device(ts.dev.shards[0].ordinal):
                tt = torch.empty((n, P), dtype=torch.float64, device="cuda")
        st, detail, failed, losses = xs.run(ts, n, tt)
        if trace:
            tr.extend(tt.cpu().numpy()[: (n if not st else failed)])
        done = n if not st else (failed if st == 5 else 0)
        ts.pipeline.advance_range(gs + 1, min(n, done + (1 if st == 5 else 0)) - 1)
        if st:
            _finish_steps(ts, done)
            _raise_step_error(ts, st, detail, f"run_steps (mini-batch {ts.global_step})")
        _finish_steps(ts, n)
        out.extend(losses)
    return np.array(out), (np.array(tr) if trace else None)


def move_est_slots(old: DeviceState, dev: DeviceState) -> None:
    """The EST context switch of an elastic rescale: every EST's slots (dropout RNG, TrackedStat)
    move from the GPU that held it to the GPU that holds it now, and executor 0's replica is copied
    to every new executor -- one 128-bit vectorised copy launch per destination GPU, reading the
    sources over NVLink (peer access), then the destinations are synchronised."""
    placement.enable_peer_access(sorted({sh.ordinal for sh in old.shards + dev.shards}))
    src0 = old.replica(0)
    for sh in dev.shards:
        pairs = []
        for osh in old.shards:  # the overlap of the old and new contiguous EST blocks
            lo, hi = max(sh.base, osh.base), min(sh.base + sh.count, osh.base + osh.count)
            if hi > lo:
                for name in ("rng", "stat_mean", "stat_count"):
                    d, o = getattr(sh, name), getattr(osh, name)
                    pairs.append((d.data_ptr() + 8 * lo, o.data_ptr() + 8 * lo, 8 * (hi - lo)))
        for j in range(len(sh.execs)):
            pairs.append((sh.replicas[j].data_ptr(), src0.data_ptr(), 2 * P * 8))
        for c in range(0, len(pairs), 64):  # (a launch takes up to 64 copy pairs)
            chunk = pairs[c:c + 64]
            dsts = (C.c_void_p * len(chunk))(*[d for d, _, _ in chunk])
            srcs = (C.c_void_p * len(chunk))(*[o for _, o, _ in chunk])
            nbytes = (C.c_int64 * len(chunk))(*[n for _, _, n in chunk])
            with torch.cuda.device(sh.ordinal):
                _native.check(_native.lib().bt_est_slot_copy(dsts, srcs, nbytes, len(chunk), stream()),
                              "EST slot copy")
    for sh in dev.shards:  # the old buffers may be freed as soon as this returns
        torch.cuda.synchronize(sh.ordinal)
    dev.invalidate()


def apply_layout(ts: TrainingState, layout: list[ExecutorSpec]) -> TrainingState:
    """Elastic restart onto a new layout, in device memory.

    Bit-for-bit the reference's checkpoint_save + checkpoint_restore
    (engine.py:332-336, checkpoint.py:204-238): contexts and one replica carry
    over; ESTs are redistributed contiguously; every new executor gets a full
    replica copy (128-bit slot-copy kernel); the bucket map is kept iff d1."""
    for ctx in ts.contexts:
        if ctx.pending_grads is not None:
            raise StateError("checkpoint requested mid-mini-batch (gradients in flight)")
        if ctx.minibatch_idx != ts.global_step:
            raise StateError("checkpoint requested mid-mini-batch (progress skew)")
    check_replica_agreement(ts)
    cfg = ts.cfg
    for spec in layout:
        cfg.kernel_profile(spec.device_kind)
    ranks = assign_ranks(list(layout), cfg.max_workers)
    old = ts.dev
    dev = DeviceState(cfg.max_workers, ranks)
    move_est_slots(old, dev)
    ex0 = ts.executors[0]
    executors = _build_executors(cfg, layout, dev, ex0._lr, ex0._mu)
    contexts = []
    for c in ts.contexts:
        nc = WorkerContext(c.virtual_rank, minibatch_idx=c.minibatch_idx)
        nc._dev = dev
        contexts.append(nc)
    dev.invalidate()
    pipe = _new_pipeline(cfg, ts.pipeline._dataset_dev)
    pipe.restore_queue(ts.pipeline.drain_for_checkpoint(), next_step=ts.global_step)
    d1 = cfg.determinism.d1
    return TrainingState(cfg, contexts, executors,
                         ts.bucket_map if d1 else build_buckets_initial(P, cfg.bucket_capacity), pipe,
                         ts.global_step, ts.epoch, rebuild_pending=not d1, dev=dev)


def reconfigure(ts: TrainingState, plan, pool) -> TrainingState:
    """Restart onto a planner configuration (engine.py:339-346).  The planner
    itself is out of scope; any object with the reference PlanConfig/DevicePool
    attributes is accepted."""
    return apply_layout(ts, plan_layout(plan, pool, ts.cfg.max_workers))


def plan_layout(plan, pool, max_workers: int) -> list[ExecutorSpec]:
    """Expand <nums, executors, threads> into executor specs (engine.py:349-376)."""
    if plan.cu_capacity < max_workers:
        raise ConfigError(f"plan capacity {plan.cu_capacity} cannot host {max_workers} workers")
    specs, remaining = [], max_workers
    for i, dtype in enumerate(pool.types):
        if plan.nums[i] > dtype.count:
            raise ConfigError(f"plan uses {plan.nums[i]} GPUs of {dtype.name!r}, pool has {dtype.count}")
        for _ in range(plan.nums[i]):
            for _ in range(plan.executors[i]):
                take = min(plan.threads[i], remaining)
                if take > 0:
                    specs.append(ExecutorSpec(dtype.name, take))
                    remaining -= take
    if remaining:
        raise ConfigError("plan layout could not host every worker")
    return specs


def executor_peak_mu(threads: int, workload_mu: float, context_mu: float = 0.75) -> float:
    """EST executor memory is flat in the EST count (engine.py:379-387)."""
    if threads < 1:
        raise ConfigError("an executor hosts at least one worker")
    return context_mu + workload_mu


def packing_peak_mu(workers: int, workload_mu: float, context_mu: float = 0.75) -> float:
    """Worker packing grows linearly (engine.py:390-395)."""
    if workers < 1:
        raise ConfigError("need at least one packed worker")
    return workers * (context_mu + workload_mu)
