"""ESCK v1 checkpoints, byte-identical to the reference's (checkpoint.py:1-238).

Little-endian layout (the reference's format doc, checkpoint.py:1-24):
  "ESCK" | u32 version=1 | u32 n, n*f64 params | f64 lr, f64 momentum,
  u32 n, n*f64 velocity | u8 d0,d1,d2 | [d1: u32 capacity, u32 nbuckets,
  per bucket u32 size + size*u32] | u32 count, per EST (u32 rank, u64 rng,
  f64 mean, u64 count, u64 minibatch_idx) | u32 count, per queued state
  (u32 worker, u32 slot, u64 rng, u64 minibatch_idx) | u64 global_step,
  u64 epoch.
`encode_esck`/`decode_esck` are pure host functions; `checkpoint_save` pulls
one replica and the EST slots from HBM, `checkpoint_restore` rebuilds the
device state on a new layout.  (In-memory elastic restarts use
engine.apply_layout, which produces the same state without the byte trip.)
"""

from __future__ import annotations

import struct

import numpy as np
import torch

from .buckets import BucketMap, build_buckets_initial
from .device import u64_to_i64
from .engine import (DeviceState, ExecutorSpec, TrainRunConfig, TrainingState, WorkerContext, _build_executors,
                     _new_pipeline, assign_ranks, check_replica_agreement)
from .errors import ConfigError, FormatError, StateError, VersionError
from .model import PARAM_COUNT
from .sampling import WorkerState

MAGIC = b"ESCK"
VERSION = 1
CONTEXT_WIRE_SIZE = struct.calcsize("<IQdQQ")  # 36 bytes per EST context


def encode_esck(doc: dict) -> bytes:
    """doc keys: params, lr, momentum, velocity, flags (d0,d1,d2), bucket_map (BucketMap|None),
    contexts [(rank, rng, mean, count, mb)], queue [(worker, slot, rng, mb)], global_step, epoch."""
    parts = [MAGIC, struct.pack("<I", VERSION)]
    params = np.asarray(doc["params"], dtype="<f8")
    vel = np.asarray(doc["velocity"], dtype="<f8")
    parts += [struct.pack("<I", params.size), params.tobytes()]
    parts += [struct.pack("<ddI", doc["lr"], doc["momentum"], vel.size), vel.tobytes()]
    d0, d1, d2 = doc["flags"]
    parts.append(struct.pack("<BBB", int(d0), int(d1), int(d2)))
    if d1:
        bm: BucketMap = doc["bucket_map"]
        parts.append(struct.pack("<II", bm.capacity, len(bm.buckets)))
        for b in bm.buckets:
            parts.append(struct.pack(f"<I{len(b)}I", len(b), *b))
    parts.append(struct.pack("<I", len(doc["contexts"])))
    parts += [struct.pack("<IQdQQ", *c) for c in doc["contexts"]]
    parts.append(struct.pack("<I", len(doc["queue"])))
    parts += [struct.pack("<IIQQ", *q) for q in doc["queue"]]
    parts.append(struct.pack("<QQ", doc["global_step"], doc["epoch"]))
    return b"".join(parts)


class _Cursor:
    def __init__(self, data: bytes):
        self.data, self.pos = data, 0

    def read(self, fmt: str):
        n = struct.calcsize(fmt)
        if self.pos + n > len(self.data):
            raise FormatError("checkpoint truncated", self.pos)
        out = struct.unpack_from(fmt, self.data, self.pos)
        self.pos += n
        return out


def decode_esck(data: bytes, cfg: TrainRunConfig | None = None) -> dict:
    """Parse and validate ESCK bytes; FormatError carries the defect's byte offset.  With `cfg`, the
    run-configuration checks fire where the reference's reader makes them (checkpoint.py:152-177):
    the determinism flags right after they are read, the context count right after it is read."""
    cur = _Cursor(bytes(data))
    (magic,) = cur.read("<4s")
    if magic != MAGIC:
        raise FormatError(f"bad magic {magic!r}", 0)
    (version,) = cur.read("<I")
    if version != VERSION:
        raise VersionError(f"unsupported checkpoint version {version}")
    (n,) = cur.read("<I")
    if n != PARAM_COUNT:
        raise FormatError(f"unexpected parameter count {n}", cur.pos - 4)
    params = list(cur.read(f"<{n}d"))
    lr, momentum = cur.read("<dd")
    (nv,) = cur.read("<I")
    if nv != n:
        raise FormatError(f"velocity count {nv} != parameter count", cur.pos - 4)
    velocity = list(cur.read(f"<{nv}d"))
    flags = tuple(bool(f) for f in cur.read("<BBB"))
    if cfg is not None and flags != (cfg.determinism.d0, cfg.determinism.d1, cfg.determinism.d2):
        raise ConfigError("checkpoint determinism flags do not match the run configuration")
    bucket_map = None
    if flags[1]:
        capacity, nb = cur.read("<II")
        buckets = []
        for _ in range(nb):
            (size,) = cur.read("<I")
            buckets.append(tuple(cur.read(f"<{size}I")))
        bucket_map = BucketMap(capacity, tuple(buckets))
        if not bucket_map.covered_exactly_once():
            raise FormatError("bucket map does not partition the parameters", cur.pos)
    (nctx,) = cur.read("<I")
    if cfg is not None and nctx != cfg.max_workers:
        raise ConfigError(f"checkpoint holds {nctx} worker contexts, run expects {cfg.max_workers}")
    contexts = [cur.read("<IQdQQ") for _ in range(nctx)]
    contexts_pos = cur.pos
    (nq,) = cur.read("<I")
    queue = [cur.read("<IIQQ") for _ in range(nq)]
    global_step, epoch = cur.read("<QQ")
    if cur.pos != len(cur.data):
        raise FormatError("trailing bytes after checkpoint payload", cur.pos)
    return {"params": params, "lr": lr, "momentum": momentum, "velocity": velocity, "flags": flags,
            "bucket_map": bucket_map, "contexts": contexts, "contexts_end": contexts_pos, "queue": queue,
            "global_step": global_step, "epoch": epoch}


def checkpoint_save(ts: TrainingState) -> bytes:
    """Serialize at a mini-batch boundary; same state -> same bytes (checkpoint.py:50-101)."""
    for ctx in ts.contexts:
        if ctx.pending_grads is not None:
            raise StateError("checkpoint requested mid-mini-batch (gradients in flight)")
        if ctx.minibatch_idx != ts.global_step:
            raise StateError("checkpoint requested mid-mini-batch (progress skew)")
    check_replica_agreement(ts)
    dev = ts.dev
    rep0 = dev.replica(0).cpu().numpy()
    rngs, means, counts = dev.snapshot()
    mode = ts.cfg.determinism
    ex0 = ts.executors[0]
    doc = {
        "params": rep0[0], "velocity": rep0[1], "lr": ex0._lr, "momentum": ex0._mu,
        "flags": (mode.d0, mode.d1, mode.d2), "bucket_map": ts.bucket_map,
        "contexts": [(c.virtual_rank, rngs[c.virtual_rank] & (2**64 - 1), means[c.virtual_rank],
                      counts[c.virtual_rank], c.minibatch_idx) for c in ts.contexts],
        "queue": [(w.worker_index, w.worker_slot, w.rng, w.minibatch_idx) for w in ts.pipeline.drain_for_checkpoint()],
        "global_step": ts.global_step, "epoch": ts.epoch,
    }
    return encode_esck(doc)


def checkpoint_restore(data: bytes, layout: list[ExecutorSpec], cfg: TrainRunConfig) -> TrainingState:
    """Rebuild a device training state on a (possibly different) layout (checkpoint.py:122-238)."""
    doc = decode_esck(data, cfg)
    mode = cfg.determinism
    if doc["flags"] != (mode.d0, mode.d1, mode.d2):
        raise ConfigError("checkpoint determinism flags do not match the run configuration")
    if len(doc["contexts"]) != cfg.max_workers:
        raise ConfigError(f"checkpoint holds {len(doc['contexts'])} worker contexts, run expects {cfg.max_workers}")
    ctx_rows = sorted(doc["contexts"], key=lambda c: c[0])
    if [c[0] for c in ctx_rows] != list(range(cfg.max_workers)):
        raise FormatError("worker contexts do not cover ranks 0..maxP-1", doc["contexts_end"])
    for spec in layout:
        cfg.kernel_profile(spec.device_kind)
    ranks = assign_ranks(list(layout), cfg.max_workers)
    dev = DeviceState(cfg.max_workers, ranks)
    dev.load_replicas(torch.tensor([doc["params"], doc["velocity"]], dtype=torch.float64))
    executors = _build_executors(cfg, layout, dev, doc["lr"], doc["momentum"])
    dev.load_contexts([u64_to_i64(c[1]) for c in ctx_rows], [c[2] for c in ctx_rows], [c[3] for c in ctx_rows])
    contexts = []
    for c in ctx_rows:
        wc = WorkerContext(c[0], minibatch_idx=c[4])
        wc._dev = dev
        contexts.append(wc)
    pipe = _new_pipeline(cfg)
    pipe.restore_queue([WorkerState(*q) for q in doc["queue"]], next_step=doc["global_step"])
    bm = doc["bucket_map"] if doc["bucket_map"] is not None else build_buckets_initial(PARAM_COUNT, cfg.bucket_capacity)
    return TrainingState(cfg, contexts, executors, bm, pipe, doc["global_step"], doc["epoch"],
                         rebuild_pending=not doc["flags"][1], dev=dev)
