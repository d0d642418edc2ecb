"""ctypes wrapper for the CPU oracle (TEST INFRASTRUCTURE ONLY).

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline /
`--impl reference` leg import this module.  The product package
(paper_2208_14228_b200) never does: it must fail loudly when its CUDA
library is missing rather than fall back to anything here.
"""

from __future__ import annotations

import ctypes as C
import os
import subprocess
from pathlib import Path

import numpy as np

HERE = Path(__file__).resolve().parent
LIB_PATH = HERE / "libbt_oracle.so"

_u64 = C.c_uint64
_i64 = C.c_int64
_dp = C.POINTER(C.c_double)
_fp = C.POINTER(C.c_float)
_u64p = C.POINTER(C.c_uint64)
_i64p = C.POINTER(C.c_int64)
_i32p = C.POINTER(C.c_int32)

OR_NUMERIC = 5


class OrCfg(C.Structure):
    _fields_ = [("seed", C.c_uint64), ("max_workers", C.c_int), ("micro_batch", C.c_int),
                ("dataset_size", C.c_int), ("lr", C.c_double), ("momentum", C.c_double),
                ("dropout_rate", C.c_double), ("jitter", C.c_double), ("bucket_capacity", C.c_int),
                ("d0", C.c_int), ("d1", C.c_int), ("d2", C.c_int), ("shuffle", C.c_int)]


def build() -> Path:
    """Compile the oracle with its Makefile (cheap; no reference sources used)."""
    subprocess.run(["make", "-s", "-C", str(HERE)], check=True)
    return LIB_PATH


_lib = None


def lib():
    global _lib
    if _lib is None:
        if not LIB_PATH.exists():
            build()
        L = C.CDLL(str(LIB_PATH))
        L.or_mix64.restype = _u64
        L.or_mix64.argtypes = [_u64]
        L.or_splitmix64_next.restype = _u64
        L.or_splitmix64_next.argtypes = [_u64p]
        L.or_derive_stream.restype = _u64
        L.or_derive_stream.argtypes = [_u64p, C.c_int]
        L.or_fnv1a64.restype = _u64
        L.or_fnv1a64.argtypes = [C.c_char_p, C.c_size_t]
        L.or_shuffled_range.argtypes = [C.c_int, _u64, _i32p]
        L.or_reduce_sum.restype = C.c_double
        L.or_reduce_sum.argtypes = [_dp, C.c_int, C.c_int]
        L.or_init_random.argtypes = [_u64, C.c_double, _dp]
        L.or_forward_backward.argtypes = [_dp, _dp, _dp, C.c_int, _i64, _u64, C.c_double, _u64, C.c_int,
                                          C.c_double, _dp, _dp, _u64p, _dp, _u64p]
        L.or_sgd_step.argtypes = [_dp, _dp, _dp, C.c_int, C.c_double, C.c_double, _dp, _dp,
                                  C.POINTER(C.c_int)]
        L.or_build_buckets_initial.argtypes = [C.c_int, C.c_int, C.POINTER(C.c_int), _i32p, _i32p]
        L.or_layout_arrival_perm.argtypes = [C.c_int, C.c_int, _u64p, _i64p, _i32p]
        L.or_allreduce.argtypes = [_dp, C.c_int, C.c_int, C.c_int, _i32p, _i32p, C.c_int, _dp]
        L.or_make_dataset.argtypes = [_u64, C.c_int, C.c_int, _dp]
        L.or_worker_rng.restype = _u64
        L.or_worker_rng.argtypes = [_u64, _u64, _u64, _u64]
        L.or_epoch_indices.argtypes = [_u64, _u64, C.c_int, C.c_int, C.c_int, C.c_int, _i32p]
        L.or_run_create.restype = C.c_void_p
        L.or_run_create.argtypes = [C.POINTER(OrCfg), C.c_int, _u64p, _i32p, _i64p]
        L.or_run_free.argtypes = [C.c_void_p]
        L.or_run_relayout.argtypes = [C.c_void_p, C.c_int, _u64p, _i32p, _i64p]
        L.or_run_step.argtypes = [C.c_void_p, _dp, _dp, _dp]
        L.or_run_set_threads.argtypes = [C.c_void_p, C.c_int]
        L.or_run_steps.argtypes = [C.c_void_p, _i64, _dp]
        L.or_run_get_state.argtypes = [C.c_void_p, _dp, _dp, _dp, _u64p, _u64p, _i64p, _i64p]
        L.or_run_get_buckets.argtypes = [C.c_void_p, _i32p, _i32p]
        L.or_reduce_update_f64.argtypes = [_dp, C.c_int, _i64, _i32p, C.c_int, _dp, _dp, C.c_double,
                                           C.c_double, _dp, _dp]
        L.or_reduce_update_f32.argtypes = [_fp, C.c_int, _i64, _i32p, C.c_int, _fp, _fp, C.c_float,
                                           C.c_float, _fp, _fp]
        L.or_reduce_update_seq_f32_mt.argtypes = [_fp, C.c_int, _i64, _fp, _fp, C.c_float, C.c_float,
                                                  _fp, _fp, C.c_int]
        L.or_libm_tanh_array.argtypes = [_dp, _i64, _dp]
        _lib = L
    return _lib


def libm_tanh(x: np.ndarray) -> np.ndarray:
    """This host's libm tanh elementwise (the reference's math.tanh, model.py:148)."""
    x = np.ascontiguousarray(x, dtype=np.float64)
    out = np.empty_like(x)
    lib().or_libm_tanh_array(_p(x, _dp), x.size, _p(out, _dp))
    return out


def _p(a: np.ndarray, t):
    return a.ctypes.data_as(t)


def fnv1a64(data: bytes) -> int:
    return lib().or_fnv1a64(data, len(data))


def mix64(x: int) -> int:
    return lib().or_mix64(x)


def splitmix64_stream(seed: int, n: int) -> list[int]:
    s = C.c_uint64(seed)
    return [lib().or_splitmix64_next(C.byref(s)) for _ in range(n)]


def derive_stream(*words: int) -> int:
    arr = (C.c_uint64 * max(1, len(words)))(*[w & (2**64 - 1) for w in words])
    return lib().or_derive_stream(arr, len(words))


def shuffled_range(n: int, state: int) -> list[int]:
    out = np.zeros(max(n, 1), dtype=np.int32)
    lib().or_shuffled_range(n, state, _p(out, _i32p))
    return out[:n].tolist()


def fanin_of(variant: str) -> int:
    return 0 if variant == "seq" else int(variant[4:])


def reduce_sum(values, variant: str) -> float:
    a = np.ascontiguousarray(values, dtype=np.float64)
    return lib().or_reduce_sum(_p(a, _dp), len(a), fanin_of(variant))


def init_random(seed: int, scale: float = 0.5) -> np.ndarray:
    out = np.zeros(161)
    lib().or_init_random(seed, scale, _p(out, _dp))
    return out


def forward_backward(params, x, y, rank, rng, stat_mean, stat_count, variant, rate):
    params = np.ascontiguousarray(params, dtype=np.float64)
    x = np.ascontiguousarray(x, dtype=np.float64)
    y = np.ascontiguousarray(y, dtype=np.float64)
    loss = C.c_double()
    grads = np.zeros(161)
    rng_o = C.c_uint64()
    mean_o = C.c_double()
    cnt_o = C.c_uint64()
    st = lib().or_forward_backward(_p(params, _dp), _p(x, _dp), _p(y, _dp), len(y), rank, rng, stat_mean,
                                   stat_count, fanin_of(variant), rate, C.byref(loss), _p(grads, _dp),
                                   C.byref(rng_o), C.byref(mean_o), C.byref(cnt_o))
    if st:
        raise ValueError(f"oracle forward_backward status {st}")
    return loss.value, grads, rng_o.value, mean_o.value, cnt_o.value


def sgd_step(params, vel, grads, lr, mu):
    params = np.ascontiguousarray(params, dtype=np.float64)
    vel = np.ascontiguousarray(vel, dtype=np.float64)
    grads = np.ascontiguousarray(grads, dtype=np.float64)
    po, vo = np.zeros_like(params), np.zeros_like(vel)
    bad = C.c_int(-1)
    st = lib().or_sgd_step(_p(params, _dp), _p(vel, _dp), _p(grads, _dp), len(params), lr, mu, _p(po, _dp),
                           _p(vo, _dp), C.byref(bad))
    if st:
        raise FloatingPointError(f"non-finite gradient at parameter {bad.value}")
    return po, vo


def buckets_initial(nparams: int, capacity: int):
    sizes = np.zeros(nparams + 1, dtype=np.int32)
    idx = np.zeros(nparams, dtype=np.int32)
    nb = C.c_int()
    lib().or_build_buckets_initial(nparams, capacity, C.byref(nb), _p(sizes, _i32p), _p(idx, _i32p))
    flat = idx.tolist()
    out, pos = [], 0
    for s in sizes[: nb.value]:
        out.append(tuple(flat[pos: pos + s]))
        pos += s
    return tuple(out)


def layout_arrival_perm(nparams: int, layout: list[tuple[str, int]]) -> list[int]:
    kf = (C.c_uint64 * len(layout))(*[fnv1a64(k.encode()) for k, _ in layout])
    th = (C.c_int64 * len(layout))(*[t for _, t in layout])
    perm = np.zeros(nparams, dtype=np.int32)
    lib().or_layout_arrival_perm(nparams, len(layout), kf, th, _p(perm, _i32p))
    return perm.tolist()


def allreduce(replicas, bucket_list, variant: str) -> np.ndarray:
    reps = np.ascontiguousarray(replicas, dtype=np.float64)
    nrep, nparams = reps.shape
    sizes = np.array([len(b) for b in bucket_list], dtype=np.int32)
    idx = np.array([i for b in bucket_list for i in b], dtype=np.int32)
    out = np.zeros(nparams)
    st = lib().or_allreduce(_p(reps, _dp), nrep, nparams, len(sizes), _p(sizes, _i32p), _p(idx, _i32p),
                            fanin_of(variant), _p(out, _dp))
    if st:
        raise ValueError(f"oracle allreduce status {st}")
    return out


def rotation_table(bucket_list, nrep: int, nparams: int) -> np.ndarray:
    """start = pos*nrep//len(bucket) per parameter (buckets.py:119-122)."""
    rot = np.zeros(nparams, dtype=np.int32)
    for b in bucket_list:
        blen = len(b)
        for pos, p in enumerate(b):
            rot[p] = pos * nrep // blen
    return rot


def reduce_update(grads: np.ndarray, rot, variant: str, params, vel, lr, mu):
    """Composite reference allreduce + sgd_step on a flat buffer (C5 checker)."""
    E, n = grads.shape
    f64 = grads.dtype == np.float64
    T, tp = (np.float64, _dp) if f64 else (np.float32, _fp)
    g = np.ascontiguousarray(grads, dtype=T)
    p_in = np.ascontiguousarray(params, dtype=T)
    v_in = np.ascontiguousarray(vel, dtype=T)
    po, vo = np.zeros_like(p_in), np.zeros_like(v_in)
    r = None if rot is None else np.ascontiguousarray(rot, dtype=np.int32)
    fn = lib().or_reduce_update_f64 if f64 else lib().or_reduce_update_f32
    st = fn(_p(g, tp), E, n, None if r is None else _p(r, _i32p), fanin_of(variant), _p(p_in, tp), _p(v_in, tp),
            lr, mu, _p(po, tp), _p(vo, tp))
    if st:
        raise FloatingPointError("non-finite synchronized gradient")
    return po, vo


def make_dataset(seed: int, n: int, dim: int = 8) -> np.ndarray:
    out = np.zeros((n, dim + 1))
    lib().or_make_dataset(seed, n, dim, _p(out, _dp))
    return out


def worker_rng(seed, epoch, local, worker) -> int:
    return lib().or_worker_rng(seed, epoch, local, worker)


def epoch_indices(seed, epoch, n, workers, micro, shuffle=True) -> list[list[int]]:
    spe = n // (workers * micro)
    out = np.zeros((workers, spe * micro), dtype=np.int32)
    st = lib().or_epoch_indices(seed, epoch, n, workers, micro, int(shuffle), _p(out, _i32p))
    if st:
        raise ValueError("bad sample plan")
    return out.tolist()


class Run:
    """Oracle restatement of init_training/run_minibatch/apply_layout for the MLP."""

    def __init__(self, seed=42, max_workers=4, micro_batch=4, dataset_size=1024, lr=0.02, momentum=0.9,
                 dropout_rate=0.5, jitter=0.1, bucket_capacity=64, mode="d1", devices=None,
                 layout=("gpu_fast",), threads=None, shuffle=True):
        mode = mode.lower()
        self.cfg = OrCfg(seed, max_workers, micro_batch, dataset_size, lr, momentum, dropout_rate, jitter,
                         bucket_capacity, 1, int("d1" in mode), int("d2" in mode), int(shuffle))
        self.devices = dict(devices or {"gpu_fast": 2, "gpu_mid": 3})
        self.E = max_workers
        self._h = None
        kf, fa, th = self._layout_args(layout, threads)
        self._h = lib().or_run_create(C.byref(self.cfg), len(layout), kf, fa, th)
        if not self._h:
            raise ValueError("oracle: invalid layout/config")

    def _layout_args(self, layout, threads):
        n = len(layout)
        kf = (C.c_uint64 * n)(*[fnv1a64(k.encode()) for k in layout])
        fa = (C.c_int32 * n)(*[self.devices[k] for k in layout])
        th = None if threads is None else (C.c_int64 * n)(*threads)
        return kf, fa, th

    def relayout(self, layout, threads=None):
        kf, fa, th = self._layout_args(layout, threads)
        st = lib().or_run_relayout(self._h, len(layout), kf, fa, th)
        if st:
            raise ValueError(f"oracle relayout status {st}")

    def set_threads(self, n: int):
        lib().or_run_set_threads(self._h, n)

    def steps(self, n: int) -> np.ndarray:
        """n pipeline-fed mini-batches in one native call; the last step's per-EST losses."""
        losses = np.zeros(self.E)
        st = lib().or_run_steps(self._h, n, losses.ctypes.data_as(_dp))
        if st:
            raise RuntimeError(f"oracle status {st}")
        return losses

    def step(self, global_batch=None) -> np.ndarray:
        losses = np.zeros(self.E)
        gx = gy = None
        if global_batch is not None:
            gb = np.ascontiguousarray(global_batch, dtype=np.float64)
            self._gx = np.ascontiguousarray(gb[:, :8])
            self._gy = np.ascontiguousarray(gb[:, 8])
            gx, gy = _p(self._gx, _dp), _p(self._gy, _dp)
        st = lib().or_run_step(self._h, gx, gy, _p(losses, _dp))
        if st == OR_NUMERIC:
            raise FloatingPointError("non-finite gradient")
        if st:
            raise ValueError(f"oracle step status {st}")
        return losses

    def state(self) -> dict:
        E = self.E
        p, v = np.zeros(161), np.zeros(161)
        sm = np.zeros(E)
        sc = np.zeros(E, dtype=np.uint64)
        rg = np.zeros(E, dtype=np.uint64)
        gs, ep = C.c_int64(), C.c_int64()
        lib().or_run_get_state(self._h, _p(p, _dp), _p(v, _dp), _p(sm, _dp), _p(sc, _u64p), _p(rg, _u64p),
                               C.byref(gs), C.byref(ep))
        return {"params": p, "velocity": v, "stat_mean": sm, "stat_count": sc, "rng": rg,
                "global_step": gs.value, "epoch": ep.value}

    def bucket_list(self):
        sizes = np.zeros(162, dtype=np.int32)
        idx = np.zeros(161, dtype=np.int32)
        nb = lib().or_run_get_buckets(self._h, _p(sizes, _i32p), _p(idx, _i32p))
        out, pos = [], 0
        for s in sizes[:nb]:
            out.append(tuple(idx[pos: pos + s].tolist()))
            pos += s
        return tuple(out)

    def __del__(self):
        if getattr(self, "_h", None):
            lib().or_run_free(self._h)
            self._h = None


def host_cores() -> int:
    return len(os.sched_getaffinity(0)) if hasattr(os, "sched_getaffinity") else os.cpu_count() or 1
