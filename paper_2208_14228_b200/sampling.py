"""Deterministic sampling and the shared data-worker pool (reference sampling.py:1-207).

Split between host and device the B200 way:
  * host (native C): the per-epoch Fisher-Yates order and round-robin deal
    (`epoch_indices`, sequential by nature), the progress-ordered queue of
    prefetched WorkerStates (pure bookkeeping, it travels in checkpoints);
  * device: the resident dataset (generated in counter form), and the
    gather + jitter of each EST's rows, fused into the step kernel's load
    (bt_mlp.cu stage A) or run standalone (`bt_jitter_gather`).
A micro-batch is a pure function of (seed, epoch, local step, EST) exactly
as in the reference, so any worker-slot count or layout yields the same bytes.
"""

from __future__ import annotations

import ctypes as C
from dataclasses import dataclass

import numpy as np
import torch

from . import _native
from .device import ptr, require_cuda, stream
from .errors import ConfigError, CorruptionError, ProgressError
from .model import INPUT_DIM
from .prng import TAG_DATA_WORKER, derive_stream

Row = tuple[tuple[float, ...], float]
_i32p = C.POINTER(C.c_int32)


def make_dataset_device(seed: int, n: int, dim: int = INPUT_DIM) -> torch.Tensor:
    """[n][dim+1] rows, all components uniform in [-1, 1) (sampling.py:24-35)."""
    require_cuda()
    out = torch.empty((n, dim + 1), dtype=torch.float64, device="cuda")
    _native.check(_native.lib().bt_make_dataset(seed & (2**64 - 1), n, dim, ptr(out), stream()), "make_dataset")
    return out


def make_dataset(seed: int, n: int, dim: int) -> list[Row]:
    rows = make_dataset_device(seed, n, dim).tolist()
    return [(tuple(r[:dim]), r[dim]) for r in rows]


@dataclass(frozen=True)
class SamplePlan:
    """One epoch's index distribution across all logical workers (drop-last)."""

    seed: int
    epoch: int
    dataset_size: int
    total_workers: int
    micro_batch: int = 1
    shuffle: bool = True

    @property
    def global_batch(self) -> int:
        return self.total_workers * self.micro_batch

    @property
    def steps_per_epoch(self) -> int:
        return self.dataset_size // self.global_batch


def epoch_indices_array(plan: SamplePlan) -> np.ndarray:
    """[workers][steps_per_epoch*micro] int32 lists (native host Fisher-Yates)."""
    if plan.total_workers < 1:
        raise ConfigError("total_workers must be >= 1")
    if plan.dataset_size < plan.total_workers:
        raise ConfigError("dataset smaller than the worker count")
    if plan.steps_per_epoch < 1:
        raise ConfigError("dataset smaller than one global batch")
    out = np.zeros((plan.total_workers, plan.steps_per_epoch * plan.micro_batch), dtype=np.int32)
    _native.check(_native.lib().bt_host_epoch_indices(plan.seed & (2**64 - 1), plan.epoch & (2**64 - 1),
                                                      plan.dataset_size, plan.total_workers, plan.micro_batch,
                                                      int(plan.shuffle), out.ctypes.data_as(_i32p)))
    return out


def epoch_indices(plan: SamplePlan) -> list[list[int]]:
    """Shuffle seeded seed^epoch, dealt round-robin (sampling.py:63-82)."""
    return epoch_indices_array(plan).tolist()


@dataclass
class WorkerState:
    """What a data worker needs to build one worker's micro-batch; the slot is metadata."""

    worker_index: int
    worker_slot: int
    rng: int
    minibatch_idx: int


def worker_rng(seed: int, epoch: int, local_step: int, worker_index: int) -> int:
    return derive_stream(TAG_DATA_WORKER, seed, epoch, local_step, worker_index)


class DataPipeline:
    """Shared data-worker pool with a progress-ordered queuing buffer."""

    EPOCH_WINDOW = 1  # epochs of index lists uploaded at least (a boundary costs one small async H2D)

    def __init__(self, seed: int, dataset_size: int, total_workers: int, micro_batch: int, jitter: float = 0.0,
                 worker_slots: int = 1, prefetch_depth: int = 2, shuffle: bool = True):
        if worker_slots < 1:
            raise ConfigError("need at least one data-worker slot")
        if prefetch_depth < 0:
            raise ConfigError("prefetch_depth must be >= 0")
        self.seed = seed
        self.dataset_size = dataset_size
        self.total_workers = total_workers
        self.micro_batch = micro_batch
        self.jitter = jitter
        self.worker_slots = worker_slots
        self.prefetch_depth = prefetch_depth
        self.shuffle = shuffle
        self.steps_per_epoch = SamplePlan(seed, 0, dataset_size, total_workers, micro_batch, shuffle).steps_per_epoch
        if self.steps_per_epoch < 1:
            raise ConfigError("dataset smaller than one global batch")
        self._dataset_dev = None
        # The queuing buffer (sampling.py:138-144, 188-197), kept lazily: the states a worker
        # prefetched itself are a pure function of their key, so only their extent is stored
        # (`_ahead[w]`: last prefetched mini-batch); states restored from a checkpoint are kept
        # verbatim in `_explicit` (they may be foreign and are checked when consumed).
        self._explicit: dict[tuple[int, int], WorkerState] = {}
        self._next_step = [0] * total_workers
        self._ahead = [-1] * total_workers
        self._lists_host: dict[int, np.ndarray] = {}
        self._lists_dev: torch.Tensor | None = None
        self._lists_dev_base = -1
        self._lists_dev_count = 0

    # ------------------------------------------------------------- device data
    @property
    def dataset_device(self) -> torch.Tensor:
        if self._dataset_dev is None:
            self._dataset_dev = make_dataset_device(self.seed, self.dataset_size, INPUT_DIM)
        return self._dataset_dev

    @property
    def dataset(self) -> list[Row]:
        rows = self.dataset_device.tolist()
        return [(tuple(r[:INPUT_DIM]), r[INPUT_DIM]) for r in rows]

    def _lists_for_epoch(self, epoch: int) -> np.ndarray:
        if epoch not in self._lists_host:
            plan = SamplePlan(self.seed, epoch, self.dataset_size, self.total_workers, self.micro_batch, self.shuffle)
            self._lists_host[epoch] = epoch_indices_array(plan)
            if len(self._lists_host) > 2 * self.EPOCH_WINDOW:
                for old in sorted(self._lists_host)[: -self.EPOCH_WINDOW]:
                    del self._lists_host[old]
        return self._lists_host[epoch]

    def _upload(self, epochs: list) -> torch.Tensor:
        """Epoch lists (host arrays) -> one device tensor [n_epochs][workers][spe*B], stream-ordered with
        no host sync: two pinned staging buffers and two device buffers used alternately (an event guards
        a staging buffer against reuse before its copy ran; a device buffer is rewritten only by a copy
        queued after every kernel that read it)."""
        per = epochs[0].size
        n = per * len(epochs)
        if getattr(self, "_stage", None) is None or self._stage[0].numel() < n:
            for p in getattr(self, "_stageptr", None) or ():  # no queued copy still reads a buffer being freed
                _native.check(_native.lib().bt_stage_wait(p), "lists staging")
            self._upload_buffers(max(n, 4 * per))
        i = self._stage_i = self._stage_i ^ 1
        if self._stage_used[i]:
            self._stage_ev[i].synchronize()
        _native.check(_native.lib().bt_stage_wait(self._stageptr[i]), "lists staging")  # a sampled call's copy
        st = self._stage_np[i]
        for k, arr in enumerate(epochs):
            st[k * per:(k + 1) * per] = arr.reshape(-1)
        _native.check(_native.lib().bt_memcpy_async(self._devptr[i], self._stageptr[i], 4 * n,
                                                    torch._C._cuda_getCurrentRawStream(torch.cuda.current_device())),
                      "lists upload")
        self._stage_ev[i].record()
        self._stage_used[i] = True
        return self._devbuf[i][:n].view(len(epochs), *epochs[0].shape)

    def lists_resident(self, first_epoch: int, last_epoch: int) -> bool:
        return (self._lists_dev is not None and self._lists_dev_base <= first_epoch
                and last_epoch < self._lists_dev_base + self._lists_dev_count)

    def reserve_lists(self, first_epoch: int, count: int) -> tuple[int, torch.Tensor]:
        """A pinned staging buffer and the device buffer that a native call (bt_mlp_run_sampled) fills with
        the lists of epochs [first_epoch, first_epoch + count) -- computed on the host inside that call;
        the pipeline then treats them as resident.  Returns (staging pointer, device view)."""
        per = self.total_workers * self.steps_per_epoch * self.micro_batch
        n = per * count
        if getattr(self, "_stage", None) is None or self._stage[0].numel() < n:
            for p in getattr(self, "_stageptr", None) or ():  # no queued copy still reads a buffer being freed
                _native.check(_native.lib().bt_stage_wait(p), "lists staging")
            self._stage = None
            self._upload_buffers(max(n, 4 * per))
        i = self._stage_i = self._stage_i ^ 1
        if self._stage_used[i]:
            self._stage_ev[i].synchronize()
        self._stage_used[i] = False  # the native call orders its own copy out of the buffer (bt_stage_wait)
        key = (i, count)  # the views are cached: a tensor view per call costs microseconds on the e2e path
        view = self._views.get(key)
        if view is None:
            view = self._views[key] = self._devbuf[i][:n].view(count, self.total_workers,
                                                               self.steps_per_epoch * self.micro_batch)
        self._lists_dev, self._lists_dev_base, self._lists_dev_count = view, first_epoch, count
        return self._stageptr[i], view

    def drop_lists(self) -> None:
        self._lists_dev = None

    def _upload_buffers(self, cap: int) -> None:
        self._stage = [torch.empty(cap, dtype=torch.int32).pin_memory() for _ in range(2)]
        self._stage_np = [t.numpy() for t in self._stage]
        self._devbuf = [torch.empty(cap, dtype=torch.int32, device="cuda") for _ in range(2)]
        self._devptr = [t.data_ptr() for t in self._devbuf]
        self._stageptr = [t.data_ptr() for t in self._stage]
        self._stage_ev = [torch.cuda.Event(), torch.cuda.Event()]
        self._stage_used = [False, False]
        self._stage_i = 0
        self._views = {}

    def device_lists(self, first_epoch: int, last_epoch: int) -> tuple[torch.Tensor, int]:
        """Resident [n_epochs][workers][spe*B] lists covering [first, last]; returns (tensor, base epoch)."""
        if not self.lists_resident(first_epoch, last_epoch):
            count = max(last_epoch - first_epoch + 1, self.EPOCH_WINDOW)
            self._lists_dev = self._upload([self._lists_for_epoch(e) for e in range(first_epoch, first_epoch + count)])
            self._lists_dev_base, self._lists_dev_count = first_epoch, count
        return self._lists_dev, self._lists_dev_base

    # ------------------------------------------------------------- bookkeeping
    def _make_state(self, step: int, worker: int) -> WorkerState:
        epoch, local = divmod(step, self.steps_per_epoch)
        slot = (step * self.total_workers + worker) % self.worker_slots
        return WorkerState(worker, slot, worker_rng(self.seed, epoch, local, worker), step)

    def _consume(self, worker: int, minibatch_idx: int) -> WorkerState:
        expected = self._next_step[worker]
        if minibatch_idx < expected:
            raise ProgressError(f"mini-batch {minibatch_idx} of worker {worker} was already consumed")
        if minibatch_idx > expected:
            raise ProgressError(f"worker {worker} must consume mini-batch {expected} before {minibatch_idx}")
        ws = self._explicit.pop((minibatch_idx, worker), None)
        if ws is not None:
            self._check_state(ws)
        else:  # prefetched earlier or made now: the same state either way
            ws = self._make_state(minibatch_idx, worker)
        self._next_step[worker] = minibatch_idx + 1
        if minibatch_idx + self.prefetch_depth > self._ahead[worker]:
            self._ahead[worker] = minibatch_idx + self.prefetch_depth
        return ws

    def _check_state(self, ws: WorkerState) -> None:
        epoch, local = divmod(ws.minibatch_idx, self.steps_per_epoch)
        if ws.rng != worker_rng(self.seed, epoch, local, ws.worker_index):
            # The device derives the worker RNG from (seed, epoch, local, EST);
            # a queued state can only differ if the checkpoint was forged.
            raise CorruptionError(f"queued worker state for ({ws.minibatch_idx}, {ws.worker_index}) has a foreign RNG")

    def batch(self, worker: int, minibatch_idx: int) -> list[Row]:
        """Produce and consume the micro-batch for (minibatch_idx, worker) (sampling.py:174-198)."""
        self._consume(worker, minibatch_idx)
        epoch, local = divmod(minibatch_idx, self.steps_per_epoch)
        lists, base = self.device_lists(epoch, epoch)
        rows = torch.empty((self.micro_batch, INPUT_DIM + 1), dtype=torch.float64, device="cuda")
        _native.check(_native.lib().bt_jitter_gather(
            ptr(self.dataset_device), ptr(lists[epoch - base]), 1, worker, self.total_workers, self.micro_batch,
            self.steps_per_epoch, self.seed & (2**64 - 1), epoch, local, float(self.jitter), ptr(rows), stream()),
            "jitter_gather")
        return [(tuple(r[:INPUT_DIM]), r[INPUT_DIM]) for r in rows.tolist()]

    def advance_all(self, minibatch_idx: int) -> None:
        """Consume (minibatch_idx, w) for every worker without producing host rows:
        the step kernel gathers them on the device.  Same progress/queue semantics as batch()."""
        nxt = self._next_step
        for w in range(self.total_workers):  # validate first so a failure leaves no partial progress
            if nxt[w] != minibatch_idx:
                self._consume(w, minibatch_idx)  # raises the reference's ProgressError
        if self._explicit:
            for w in range(self.total_workers):
                self._consume(w, minibatch_idx)
            return
        self._next_step = [minibatch_idx + 1] * self.total_workers
        ahead = minibatch_idx + self.prefetch_depth
        self._ahead = [a if a > ahead else ahead for a in self._ahead]

    def advance_range(self, first: int, count: int) -> None:
        """advance_all for mini-batches first .. first+count-1 (one persistent launch's worth)."""
        if self._explicit or count < 1 or any(n != first for n in self._next_step):
            for k in range(count):
                self.advance_all(first + k)
            return
        self._next_step = [first + count] * self.total_workers
        ahead = first + count - 1 + self.prefetch_depth
        self._ahead = [a if a > ahead else ahead for a in self._ahead]

    def drain_for_checkpoint(self) -> list[WorkerState]:
        """Every queued state in (mini-batch, worker) order (sampling.py:200-202)."""
        q = dict(self._explicit)
        for w in range(self.total_workers):
            for step in range(self._next_step[w], self._ahead[w] + 1):
                if (step, w) not in q:
                    q[(step, w)] = self._make_state(step, w)
        return [q[k] for k in sorted(q)]

    def restore_queue(self, states: list[WorkerState], next_step: int) -> None:
        self._explicit = {(ws.minibatch_idx, ws.worker_index): ws for ws in states}
        self._next_step = [next_step] * self.total_workers
        self._ahead = [-1] * self.total_workers
