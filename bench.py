"""Benchmark of the deterministic elastic-DP step (BASELINE.json metric).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl b200|reference]

Workload (BASELINE.json configs[1], "C2"): the reference MLP, 8 ESTs x
micro-batch 4 (32 samples per mini-batch), seed 42, 1024-row synthetic
dataset, d1, Tree(2) device kind, momentum SGD; a "step" is one mini-batch.

* value  -- samples/s with everything resident in HBM: the fused persistent
  step kernel (bt_mlp.cu), timed with CUDA events on its stream; the K steps
  run as launches of 100 mini-batches (C2's 100-step run) each, with an L2
  flush (256 MiB write) between launches, outside the timed spans.
* e2e    -- the same K mini-batches through the C-ABI with HOST buffers: each
  launch's global batches (split_by_rank rows) are copied from pinned host
  memory and its per-EST losses copied back inside the timed span.
* roofline -- the step kernel (latency-bound: 32 samples/step), plus the
  deterministic reducer (bt_reduce.cu, C5 shape) measured against HBM, and the
  deterministic tcgen05 GEMM (bt_gemm.cu, 8192^3 bf16) against the tensor peak.
* cpu_baseline -- the CPU oracle (a C restatement of the reference) on a
  bounded sample of the same workload, on this box's host cores.
N > 1 (torchrun): the 8 ESTs are split into contiguous rank blocks; each rank
runs its ESTs' forward/backward, the EST gradient slots are exchanged with an
NCCL all-gather (a bit copy), and every rank applies the same fixed-order
reduce + SGD kernel, so all ranks hold bit-identical weights ("scaling":
"strong": the job's total work is fixed).
"""

from __future__ import annotations

import argparse
import ctypes as C
import json
import os
import statistics
import subprocess
import sys
import time
from pathlib import Path

import numpy as np
import torch

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

METRIC = "samples/sec at 1/2/4/8 B200 with bit-identical weights across mappings"
E_TOTAL, MICRO, NROWS, SEED = 8, 4, 1024, 42
SAMPLES_PER_STEP = E_TOTAL * MICRO
LAUNCH = 100  # mini-batches per timed launch (C2 is a 100-step run)
PEAKS = {"hbm_gbs": 6541.8, "bf16_tflops": 1639.6, "bf16_tflops_sustained": 1358.3}


def load_peaks():
    p = ROOT / "MEASURED_PEAKS.json"
    if p.exists():
        try:
            d = json.loads(p.read_text())
            return {k: d.get(k, v) for k, v in PEAKS.items()}, "measured"
        except Exception:
            pass
    return {"hbm_gbs": 6650.0, "bf16_tflops": 1590.0, "bf16_tflops_sustained": 1400.0}, "fallback"


class ClockSampler:
    """nvidia-smi clocks + throttle reasons sampled while the benchmark runs."""

    FIELDS = ("clocks.sm,clocks.max.sm,clocks_event_reasons.active,clocks_event_reasons.hw_slowdown,"
              "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
              "clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int):
        self.proc = None
        try:
            self.proc = subprocess.Popen(["nvidia-smi", "-i", str(index), f"--query-gpu={self.FIELDS}",
                                          "--format=csv,noheader,nounits", "-lms", "100"],
                                         stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
        except OSError:
            self.proc = None
        self.busy = []
        self.first = ""
        if self.proc is not None:  # let nvidia-smi finish starting up (driver queries) before anything is timed
            import select

            if select.select([self.proc.stdout], [], [], 15.0)[0]:
                self.first = self.proc.stdout.readline()
            time.sleep(0.2)

    def mark(self):
        self.busy.append(time.time())

    def stop(self) -> dict:
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        self.proc.terminate()
        out, _ = self.proc.communicate(timeout=10)
        out = self.first + out
        sm, smax, reasons = [], [], set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for line in out.strip().splitlines():
            f = [x.strip() for x in line.split(",")]
            if len(f) < 7:
                continue
            try:
                sm.append(float(f[0]))
                smax.append(float(f[1]))
            except ValueError:
                continue
            for n, v in zip(names, f[3:7]):
                if v.lower() == "active":
                    reasons.add(n)
        loaded = [s for s in sm if s > 0.5 * max(sm)] if sm else []
        return {"sm_mhz": statistics.median(loaded) if loaded else None,
                "sm_max_mhz": max(smax) if smax else None, "reasons": sorted(reasons), "samples": len(sm)}


def ncu_traffic(kernel: str):
    """dram__bytes_read.sum + dram__bytes_write.sum of one launch, from the committed
    `ncu --set full` capture summarised in profiles/ (tools/summarize_ncu.py)."""
    p = ROOT / "profiles" / "traffic.json"
    try:
        return json.loads(p.read_text()).get(kernel)
    except (OSError, ValueError):
        return None


def _native_lib():
    from paper_2208_14228_b200 import _native

    return _native.lib()


class HostGate:
    """Holds a stream at a device-side wait on a pinned host word until the host has enqueued the
    whole timed region, so the CUDA-event span holds the kernels only -- not host scheduling jitter
    between the first event and the launch (cuStreamWaitValue32 on mapped host memory)."""

    # Under a profiler that serialises launches (Nsight Compute: its injection sets NV_TPS_LAUNCH_TOKEN /
    # NV_NSIGHT_INJECTION_*) a kernel queued behind the gate would wait for a host write that only comes
    # after its launch call returns: the gate is then a no-op (profiled runs are never bench values).
    PASS = any(k in os.environ for k in ("NV_TPS_LAUNCH_TOKEN", "NV_NSIGHT_INJECTION_TRANSPORT_TYPE",
                                         "CUDA_INJECTION64_PATH")) or os.environ.get("BT_BENCH_GATE") == "0"

    def __init__(self):
        self.word = torch.zeros(1, dtype=torch.int32).pin_memory()
        self.np = self.word.numpy()
        self.n = 0

    def close(self, stream) -> None:
        from paper_2208_14228_b200 import _native

        if self.PASS:
            return
        self.n += 1
        _native.check(_native.lib().bt_stream_wait_u32_geq(self.word.data_ptr(), self.n, stream.cuda_stream),
                      "host gate")

    def open(self) -> None:
        self.np[0] = self.n


# ------------------------------------------------------------------ b200 arm
def make_cfg(bt):
    return bt.TrainRunConfig(seed=SEED, max_workers=E_TOTAL, micro_batch=MICRO, dataset_size=NROWS, lr=0.02,
                             momentum=0.9, dropout_rate=0.5, jitter=0.1, bucket_capacity=64,
                             determinism=bt.DeterminismMode.from_label("d1"),
                             device_fanins={"gpu_fast": 2, "gpu_mid": 3})


def chunks(K: int, spe: int):
    out, left = [], K
    while left > 0:
        out.append(min(spe, left))
        left -= out[-1]
    return out


def bench_device_single(bt, K: int, W: int, flush):
    """N=1, inputs resident in HBM: the fused persistent kernel, one launch per chunk of at most
    LAUNCH mini-batches (the prepared launch of run_steps, engine._FastStep), CUDA events on its
    stream around each launch, L2 flushed before each launch (outside the span)."""
    from paper_2208_14228_b200 import _native, engine

    cfg = make_cfg(bt)
    ts = bt.init_training(cfg, [bt.ExecutorSpec("gpu_fast")])
    for n in chunks(W, LAUNCH):
        engine.run_steps(ts, n)
    torch.cuda.synchronize()
    fs = engine._fast(ts)
    gate = HostGate()
    spans = []
    launches = 0
    s = torch.cuda.current_stream()
    for n in chunks(K, LAUNCH):
        ts.pipeline.advance_range(ts.global_step, n)
        gs, spe = ts.global_step, ts.pipeline.steps_per_epoch
        lists, base = ts.pipeline.device_lists(gs // spe, (gs + n - 1) // spe)
        a = fs.a
        a.K, a.step0, a.lists, a.epoch_base = n, gs, lists.data_ptr(), base
        a.losses = fs.io_ptr + 8 * (fs.KMAX - n) * fs.E  # the launch's rows of the shard's I/O block
        flush()
        gate.close(s)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        try:
            e0.record(s)
            _native.check(_native.lib().bt_mlp_step(C.byref(a), s.cuda_stream))
            e1.record(s)
        finally:
            gate.open()
        launches += 1
        e1.synchronize()
        spans.append(e0.elapsed_time(e1))
        st_, _, _ = ts.dev.flags.status()
        assert st_ == 0, st_
        engine._finish_steps(ts, n)
        ts.dev.invalidate()
    return ts, sum(spans), spans, launches, a.est_per_cta


def bench_e2e_single(bt, K: int, W: int, flush):
    """N=1 end to end through the public API (engine.run_steps, the K-mini-batch form of
    run_minibatch), timed on the host clock: every launch starts from HOST inputs -- the epoch
    index lists are recomputed (native Fisher-Yates, the reference's sampling.py:63-82) and copied
    host->device inside the span -- and returns HOST outputs (per-EST losses + status, device->host,
    stream synchronised) inside the span.  L2 flushed before each launch (outside the span)."""
    from paper_2208_14228_b200 import engine

    cfg = make_cfg(bt)
    ts = bt.init_training(cfg, [bt.ExecutorSpec("gpu_fast")])
    pipe = ts.pipeline
    # W warm-up mini-batches, one call each and prepared like a timed call: the host / driver / launch path
    # of a call is warmed W times (its first calls in a process run 1.5-2x slower: tools/e2e_first_call.py)
    for _ in range(W):
        flush()
        pipe._lists_dev = None
        pipe._lists_host.clear()
        torch.cuda.synchronize()
        engine.run_steps(ts, 1)
    torch.cuda.synchronize()
    spans, launches, h2d, d2h = [], 0, 0, 0
    losses = []
    for n in chunks(K, LAUNCH):
        flush()
        pipe._lists_dev = None   # nothing of the inputs stays resident between launches
        pipe._lists_host.clear()
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        out, _ = engine.run_steps(ts, n)
        spans.append((time.perf_counter() - t0) * 1e3)
        launches += 1
        h2d += pipe._lists_dev.numel() * 4
        d2h += out.size * 8 + 16
        losses.append(out)
    return ts, sum(spans), launches, h2d / K, d2h / K, np.concatenate(losses)


def bench_run_minibatch(bt, calls: int = 300, warm: int = 30):
    """The reference API's per-step call (run_minibatch: one mini-batch, host losses back), wall
    clock per call, median over `calls` calls."""
    cfg = make_cfg(bt)
    ts = bt.init_training(cfg, [bt.ExecutorSpec("gpu_fast")])
    for _ in range(warm):
        bt.run_minibatch(ts)
    times = []
    for _ in range(calls):
        t0 = time.perf_counter()
        bt.run_minibatch(ts)
        times.append((time.perf_counter() - t0) * 1e6)
    return {"us_per_call": round(statistics.median(times), 2), "p10_us": round(sorted(times)[calls // 10], 2),
            "p90_us": round(sorted(times)[calls * 9 // 10], 2), "calls": calls,
            "samples_per_s": round(SAMPLES_PER_STEP / (statistics.median(times) / 1e6), 1)}


def bench_device_dist(bt, K: int, W: int, rank: int, world: int, flush, e2e: bool, exchange: str):
    """N>1: EST blocks per rank (paper_2208_14228_b200.dist.DistributedTrainer).

    exchange "xdev" (default): the persistent lock-step kernel -- each rank runs a chunk of up to
    LAUNCH mini-batches in one launch and exchanges EST slots every mini-batch through the other
    ranks' inboxes (CUDA IPC peer memory, device-side counters).  Device spans: every rank holds
    its stream at a host gate, queues [e0, launch, e1], all ranks meet at a host barrier, then the
    gates open together -- the span is the lock-step kernel, not launch skew between processes.
    e2e: host clock around the chunk on every rank (the epoch lists recomputed on the host and
    uploaded, the launch, the losses and status copied back, the stream synchronised), max over
    ranks by the caller.
    exchange "ipc" / "allgather": the per-mini-batch grads-only kernel + reducer paths."""
    import torch.distributed as dist

    from paper_2208_14228_b200.dist import DistributedTrainer

    tr = DistributedTrainer(seed=SEED, max_workers=E_TOTAL, micro_batch=MICRO, dataset_size=NROWS,
                            exchange=None if exchange == "xdev" else exchange)
    spe = tr.pipe.steps_per_epoch
    s = torch.cuda.current_stream()
    spans, h2d, d2h, launches = [], 0, 0, 0
    if tr.exchange == "xdev":
        for n in chunks(W, LAUNCH):
            tr.run(n)
        torch.cuda.synchronize()
        dist.barrier()
        gate = HostGate()
        host_out = torch.empty((LAUNCH, E_TOTAL), dtype=torch.float64).pin_memory()
        host_st = torch.zeros(4, dtype=torch.int32).pin_memory()
        for n in chunks(K, LAUNCH):
            flush()
            if e2e:
                tr.pipe._lists_dev = None  # nothing of the inputs stays resident between launches
                tr.pipe._lists_host.clear()
                torch.cuda.synchronize()
                dist.barrier()
                t0 = time.perf_counter()
                out = tr.run(n)
                host_out[:n].copy_(out, non_blocking=True)
                host_st.copy_(tr.flags.t, non_blocking=True)
                s.synchronize()
                spans.append((time.perf_counter() - t0) * 1e3)
                h2d += tr._xlists.numel() * 4
                d2h += n * tr.count * 8 + 16
                assert int(host_st[0]) == 0, int(host_st[0])
            else:
                gate.close(s)
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                try:
                    e0.record(s)
                    tr.run(n)
                    e1.record(s)
                    dist.barrier()
                finally:
                    gate.open()
                e1.synchronize()
                spans.append(e0.elapsed_time(e1))
            launches += 1
        tr.check()
        torch.cuda.synchronize()
        dist.barrier()
        params = tr.params[0].clone()
        tr.close()
        return params, sum(spans), launches, h2d / K, d2h / K
    host_losses = torch.empty((K + W, tr.count), dtype=torch.float64).pin_memory()
    for _ in range(W):
        tr.step()
    torch.cuda.synchronize()
    dist.barrier()
    for n in chunks(K, spe):
        if e2e:
            tr.pipe._lists_dev = None  # force the epoch's lists through host memory again
        flush()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(s)
        for _ in range(n):
            step = tr.step_idx
            losses = tr.step()
            if e2e:
                host_losses[step].copy_(losses, non_blocking=True)
        e1.record(s)
        e1.synchronize()
        spans.append(e0.elapsed_time(e1))
        if e2e:
            h2d += tr.pipe._lists_dev.numel() * 4
    tr.check()
    dist.barrier()
    return tr.params[0].clone(), sum(spans), 2 * K, h2d / K, tr.count * 8


def bench_reducer(flush, peaks, E=8, S_MB=256, iters=10):
    """C5-shaped deterministic reducer, G=1: E f32 EST gradient slots of S MB each,
    RankTree(2) order, fused /E + momentum SGD.  HBM_alg = E*S + 4*S bytes."""
    from paper_2208_14228_b200 import _native
    from paper_2208_14228_b200.device import Flags, stream

    n = S_MB * 2**20 // 4
    g = torch.empty((E, n), dtype=torch.float32, device="cuda").uniform_(-1, 1)
    p = torch.empty(n, dtype=torch.float32, device="cuda").uniform_(-1, 1)
    v = torch.zeros(n, dtype=torch.float32, device="cuda")
    flags = Flags()
    out = {}
    for name, fan in (("rank_tree2", 2), ("sequential", 0)):
        a = _native.ReduceArgs()
        a.dtype, a.mode, a.E, a.fanin, a.n = _native.DTYPE_F32, _native.REDUCE_UPDATE, E, fan, n
        for k in range(E):
            a.grads[k] = g[k].data_ptr()
        a.param, a.vel, a.param_out, a.vel_out = p.data_ptr(), v.data_ptr(), p.data_ptr(), v.data_ptr()
        a.lr, a.mu, a.flags = 1e-9, 0.9, flags.t.data_ptr()
        for _ in range(2):
            _native.check(_native.lib().bt_reduce_update(C.byref(a), stream()))
        times = []
        s = torch.cuda.current_stream()
        for _ in range(iters):
            flush()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(s)
            _native.check(_native.lib().bt_reduce_update(C.byref(a), stream()))
            e1.record(s)
            e1.synchronize()
            times.append(e0.elapsed_time(e1))
        ms = statistics.median(times)
        alg = (E + 4) * n * 4
        out[name] = {"ms": ms, "achieved_gbs": alg / ms / 1e6, "frac": alg / ms / 1e6 / peaks["hbm_gbs"]}
    del g, p, v
    torch.cuda.empty_cache()
    best = out["rank_tree2"]
    return {"kernel": "reduce_fast_kernel<float,8,2> (bt_reduce.cu)", "E": E, "S_MB": S_MB, "dtype": "f32",
            "traffic": ncu_traffic("reduce_fast_kernel"),
            "bound": "hbm", "achieved": round(best["achieved_gbs"], 1), "peak": peaks["hbm_gbs"], "unit": "GB/s",
            "frac": round(best["frac"], 4), "bytes_per_launch": (E + 4) * n * 4, "ms": round(best["ms"], 4),
            "variants": {k: {kk: round(vv, 4) for kk, vv in d.items()} for k, d in out.items()}}


def bench_reducer_dist(rank: int, world: int, dist, peaks, E=64, S_MB=256, iters=5):
    """C5 on N GPUs: the guarded peer-memory reducer (paper_2208_14228_b200/peer.py,
    RankTree(2)) -- each rank folds its E/N EST slots of S MB (f32) into a subtree partial in HBM, the owner
    of each parameter shard folds the N partials with NVLink peer loads, checks, applies momentum SGD and
    stores its shard into every replica.  Time = CUDA events on each rank's reducer stream between host
    barriers, max over ranks.  NVLink_alg = 2 (N-1)/N S per direction per GPU (partials in, shard out);
    HBM_alg per GPU = (E/N + 1) S (subtree) + ~(N + 6) S/N (owner: partials, param, velocity, staging)."""
    from paper_2208_14228_b200.hier import RankBuffers
    from paper_2208_14228_b200.peer import PeerGroupReducer

    n = S_MB * 2**20 // 4
    E_loc = E // world
    st = torch.cuda.Stream()
    g = torch.empty((E_loc, n), dtype=torch.float32, device="cuda").uniform_(-1e-3, 1e-3)
    loc = RankBuffers(g, torch.zeros(n, dtype=torch.float32, device="cuda"),
                      torch.zeros(n, dtype=torch.float32, device="cuda"), st)
    red = PeerGroupReducer(loc, E, "rank_tree2", None, 1e-9, 0.9)
    times = []
    for it in range(iters + 2):
        torch.cuda.synchronize()
        dist.barrier()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(st)
        red.step()
        e1.record(st)
        e1.synchronize()
        if it >= 2:
            times.append(e0.elapsed_time(e1))
    red.check()
    t = torch.tensor([statistics.median(times)], dtype=torch.float64, device="cuda")
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    ms = float(t.item())
    red.close()
    del g, loc, red
    torch.cuda.empty_cache()
    S = S_MB * 2**20
    nvl = 2.0 * (world - 1) / world * S
    hbm = (E_loc + 1) * S + (world + 6) * S / world
    nvl_peak = 900.0  # GB/s per direction per GPU (NVLink 5 / NVSwitch)
    t_min = max(hbm / peaks["hbm_gbs"] / 1e6, nvl / nvl_peak / 1e6)
    return {"kernel": "reduce_fast_kernel (subtree) + owner fold over NVLink peer loads (peer.PeerGroupReducer, "
                      "RankTree(2), guarded)", "E": E, "S_MB": S_MB, "n_gpus": world, "dtype": "f32",
            "ms": round(ms, 4), "nvlink_alg_bytes_per_dir": int(nvl), "hbm_alg_bytes": int(hbm),
            "nvlink_gbs": round(nvl / ms / 1e6, 1), "nvlink_peak_gbs": nvl_peak,
            "hbm_gbs": round(hbm / ms / 1e6, 1), "hbm_peak_gbs": peaks["hbm_gbs"],
            "frac_of_roofline": round(t_min / ms, 4), "roofline_ms": round(t_min, 4),
            "bound": "nvlink" if nvl / nvl_peak > hbm / peaks["hbm_gbs"] else "hbm"}


def bench_gemm(flush, peaks, M=8192, N=8192, K=8192, iters=10):
    """SURVEY §8f row 2 brick: the deterministic tcgen05 GEMM (bt_gemm.cu) at 8192^3 bf16 -> bf16,
    against the measured bf16 tensor peak, with cuBLAS (torch.matmul) on the same shape beside it."""
    from paper_2208_14228_b200.gemm import gemm_bf16

    a = torch.randn(M, K, device="cuda").to(torch.bfloat16)
    b = torch.randn(N, K, device="cuda").to(torch.bfloat16)
    s = torch.cuda.current_stream()

    def med(fn):
        for _ in range(2):
            fn()
        times = []
        for _ in range(iters):
            flush()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(s)
            fn()
            e1.record(s)
            e1.synchronize()
            times.append(e0.elapsed_time(e1))
        return statistics.median(times)

    ms = med(lambda: gemm_bf16(a, b, torch.bfloat16))
    ms_cublas = med(lambda: torch.matmul(a, b.T))
    again = gemm_bf16(a, b, torch.bfloat16, grid=37)  # bits independent of the grid (determinism)
    same = bool(torch.equal(gemm_bf16(a, b, torch.bfloat16).view(torch.int16), again.view(torch.int16)))
    fl = 2.0 * M * N * K
    del a, b, again
    torch.cuda.empty_cache()
    tf = fl / ms / 1e9
    return {"kernel": "gemm_bf16_tn_pair_kernel<5,bf16> (bt_gemm.cu: tcgen05 cta_group::2 + TMA, 256x256 tile per CTA pair, fixed K order)",
            "shape": [M, N, K], "bound": "tensor", "achieved": round(tf, 1), "peak": peaks["bf16_tflops"],
            "unit": "TFLOP/s", "frac": round(tf / peaks["bf16_tflops"], 4), "ms": round(ms, 4),
            "traffic": ncu_traffic("gemm_bf16_tn_kernel"), "cublas_tflops": round(fl / ms_cublas / 1e9, 1),
            "grid_invariant_bits": same}


def bench_bert(peaks, ests=32, steps=5, warmup=3):
    """C4 (BASELINE.json configs[3]): BERT-base encoder (12 x 768, 12 heads, FFN 3072, seq 128, dropout 0.1),
    32 ESTs x 8 sequences, deterministic tcgen05 GEMMs + fixed-order reducer (paper_2208_14228_b200/bert.py).
    Step time by CUDA events; per-kernel split of one step by CUPTI (torch.profiler); the same 32 ESTs as
    4 launch groups of 8 (the 4-GPU mapping's per-GPU work) must give bit-identical weights."""
    from torch.profiler import ProfilerActivity, profile

    from paper_2208_14228_b200.bert import BertJob

    job = BertJob(ests=ests, est_group=4, fanin=2)
    s = torch.cuda.current_stream()
    for _ in range(warmup):
        job.step()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(s)
    for _ in range(steps):  # the non-finite check once after the timed steps (the update is guarded on device)
        losses = job.step(check=False)
    e1.record(s)
    e1.synchronize()
    job.check_status()
    ms = e0.elapsed_time(e1) / steps
    with profile(activities=[ProfilerActivity.CUDA]) as prof:
        job.step()
        torch.cuda.synchronize()
    split = {}
    for ev in prof.events():
        if ev.device_type == torch.autograd.DeviceType.CUDA:
            key = next((k for k in ("gemm_bf16", "attn_fwd", "attn_bwd", "ln_fwd", "ln_bwd", "reduce", "colsum",
                                    "cast_t", "embed", "ce_kernel", "sort_segments") if k in ev.name), "other")
            split[key] = split.get(key, 0.0) + ev.device_time_total / 1e3
    import paper_2208_14228_b200 as bt

    fnv_one = f"{bt.fnv1a64(job.params.cpu().numpy().tobytes()):016x}"
    flops = job.gemm_flops_per_step()
    # the dominant kernel, per launch: the FFN forward GEMM (T x 3072 x 768, bias + GELU epilogue), timed
    # alone on its stream with CUDA events (inputs: layer 0's activations of the last step)
    from paper_2208_14228_b200 import _native
    from paper_2208_14228_b200.device import stream as cur_stream

    w, L = job._workspace(ests)["layers"][0], _native.lib()
    T, D, F = ests * job.Te, job.D, job.F

    def ffn_gemm():
        _native.check(L.bt_gemm_bf16_ffn(w["h1b"].data_ptr(), job._wb(0, "W1"), w["Hpre"].data_ptr(), T, F, D, 1,
                                         job._p(0, "b1"), None, w["Dact"].data_ptr(), 42, 0, 0, job.Te, 0.0, 0,
                                         cur_stream()))
    for _ in range(3):
        ffn_gemm()
    g0, g1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    g0.record(s)
    for _ in range(20):
        ffn_gemm()
    g1.record(s)
    g1.synchronize()
    ffn_ms = g0.elapsed_time(g1) / 20
    ffn_tf = 2.0 * T * F * D / ffn_ms / 1e9
    del job
    torch.cuda.empty_cache()
    per_est = BertJob(ests=ests, fanin=2)  # one gradient buffer per EST (est_group 1)
    for _ in range(warmup):
        per_est.step()
    torch.cuda.synchronize()
    e0.record(s)
    for _ in range(steps):
        per_est.step()
    e1.record(s)
    e1.synchronize()
    ms_per_est = e0.elapsed_time(e1) / steps
    del per_est
    torch.cuda.empty_cache()
    from paper_2208_14228_b200.runlog import bitdiff

    a, b = BertJob(ests=ests, layers=2, est_group=4, fanin=2), BertJob(ests=ests, layers=2, est_group=4, fanin=2)
    la, lb = a.run_log(2), b.run_log(2, groups=[ests // 4] * 4)  # per-EST losses + weight fingerprints per step
    same = bool(torch.equal(a.params.view(torch.int32), b.params.view(torch.int32))) and bitdiff(la, lb) is None
    grouping_fp = la.records[-1].param_hash
    del a, b
    torch.cuda.empty_cache()
    gemm_ms = split.get("gemm_bf16", 0.0)
    seqs = ests * 8
    return {"workload": "C4: BERT-base bf16 (token ids from splitmix64 mod 30522, word + position embeddings, 12 "
                        "layers, d 768, 12 heads, FFN 3072, seq 128, dropout 0.1 hidden + attention, masked-LM head "
                        "tied to the word embedding: 20 masked positions per sequence, cross-entropy over the "
                        "vocabulary), 32 ESTs x 8 sequences, momentum SGD (BASELINE.json configs[3]); gradient leaves "
                        "of 4 ESTs (EST-ordered accumulation, valid for 1/2/4/8 GPUs), Tree(2) reducer",
            "samples_per_s": round(seqs / (ms / 1e3), 1), "unit": "sequences/s", "ms_per_step": round(ms, 3),
            "per_est_gradient_buffers": {"samples_per_s": round(seqs / (ms_per_est / 1e3), 1),
                                         "ms_per_step": round(ms_per_est, 3)},
            "tokens_per_s": round(seqs * 128 / (ms / 1e3), 1), "loss": round(losses.mean().item(), 5),
            "roofline": {"kernel": "gemm_bf16_tn_pair_kernel<5,bf16> FFN forward (bt_gemm.cu: 32768x3072x768, "
                                   "bias+GELU epilogue, TMA-store), one launch",
                         "bound": "tensor", "achieved": round(ffn_tf, 1), "peak": peaks["bf16_tflops"],
                         "unit": "TFLOP/s", "frac": round(ffn_tf / peaks["bf16_tflops"], 4),
                         "ms": round(ffn_ms, 4), "traffic": ncu_traffic("bert_ffn_gemm"),
                         "all_step_gemms_tflops": round(flops / gemm_ms / 1e9, 1) if gemm_ms else None,
                         "step_level_tflops": round(flops / ms / 1e9, 1), "dense_flops_per_step": flops,
                         "note": "L2 not flushed between the 20 back-to-back launches (55 MB of operands)"},
            "kernel_ms_per_step": {k: round(v, 3) for k, v in sorted(split.items(), key=lambda kv: -kv[1])},
            "bit_identical_groupings": {"groups": [[ests], [ests // 4] * 4], "layers": 2, "steps": 2, "equal": same,
                                        "run_logs": "runlog.bitdiff: no divergence", "weights_fp": grouping_fp},
            "params_fnv": fnv_one}


def replicas_identical(dist, data: bytes) -> tuple[bool, str]:
    """Byte-level agreement of every rank's replica: FNV-1a of the bytes gathered from every rank
    and the bytes themselves compared against rank 0's (no checksum that cancels)."""
    import paper_2208_14228_b200 as bt

    h = f"{bt.fnv1a64(data):016x}"
    hs = [None] * dist.get_world_size()
    dist.all_gather_object(hs, h)
    blobs = [None] * dist.get_world_size()
    dist.all_gather_object(blobs, data)
    return len(set(hs)) == 1 and all(b == blobs[0] for b in blobs), h


def bench_bert_dist(rank, world, dist, ests=32, steps=5, warmup=3, **model):
    """C4 on N GPUs: rank r holds ESTs [r*E/N, (r+1)*E/N) and exchanges through the peer-memory reducer
    (RankTree(2): subtree partials + NVLink owner fold, fused /E + SGD, updated shards stored into every
    replica).  Step time = max over ranks (CUDA events); replicas must agree bitwise."""
    from paper_2208_14228_b200.bert import BertJob

    n = ests // world
    job = BertJob(ests=ests, est_base=rank * n, est_count=n, fanin=2, est_group=min(4, n), **model)
    dev = "cuda" if dist.get_backend() == "nccl" else "cpu"  # gloo: host tensors (tests)
    job.attach_peer()
    s = torch.cuda.current_stream()
    for _ in range(warmup):
        job.step()
    torch.cuda.synchronize()
    dist.barrier()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(s)
    for _ in range(steps):  # the non-finite check once after the timed steps (the update is guarded on device)
        job.step(check=False)
    e1.record(s)
    e1.synchronize()
    job.check_status()
    t = torch.tensor([e0.elapsed_time(e1) / steps], dtype=torch.float64, device=dev)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    ms = t.item()
    same, h = replicas_identical(dist, job.params.cpu().numpy().tobytes())
    torch.cuda.synchronize()
    dist.barrier()
    job.peer.close()
    del job
    torch.cuda.empty_cache()
    return {"workload": "C4: BERT-base encoder bf16, 32 ESTs x 8 sequences, EST blocks per GPU, peer-memory "
                        "RankTree(2) reducer (BASELINE.json configs[3])",
            "samples_per_s": round(ests * model.get("seqs", 8) / (ms / 1e3), 1), "unit": "sequences/s",
            "ms_per_step": round(ms, 3), "n_gpus": world, "ests_per_gpu": n, "replicas_bit_identical": same, "params_fnv": h}


def bench_resnet_dist(rank, world, dist, ests=16, batch=32, steps=10, warmup=3):
    """C3 on N GPUs: rank r holds ESTs [r*E/N, (r+1)*E/N) (their BN slots and cursors), peer-memory
    Tree(2) reducer; step time = max over ranks; replicas must agree bitwise."""
    from paper_2208_14228_b200.resnet import ResNetJob

    n = ests // world
    job = ResNetJob(ests=ests, batch=batch, gpus=1, est_base=rank * n, est_count=n, fanin=2)
    job.attach_peer()
    dev = "cuda" if dist.get_backend() == "nccl" else "cpu"
    s = torch.cuda.current_stream()
    for _ in range(warmup):
        job.step()
    torch.cuda.synchronize()
    dist.barrier()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(s)
    for _ in range(steps):  # the non-finite check once after the timed steps (the update is guarded on device)
        job.step(check=False)
    e1.record(s)
    e1.synchronize()
    job.check_status()
    t = torch.tensor([e0.elapsed_time(e1) / steps], dtype=torch.float64, device=dev)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    ms = t.item()
    same, h = replicas_identical(dist, job.params.cpu().numpy().tobytes())
    torch.cuda.synchronize()
    dist.barrier()
    job.peer.close()
    del job
    torch.cuda.empty_cache()
    return {"workload": "C3: ResNet-18 with per-EST BatchNorm, 16 ESTs x 32 images, EST blocks (and their BN slots) "
                        "per GPU, peer-memory RankTree(2) reducer (BASELINE.json configs[2])",
            "samples_per_s": round(ests * batch / (ms / 1e3), 1), "unit": "images/s", "ms_per_step": round(ms, 3),
            "n_gpus": world, "ests_per_gpu": n, "replicas_bit_identical": same, "params_fnv": h}


def bench_resnet(peaks, ests=16, batch=32, steps=10, warmup=3):
    """C3 (BASELINE.json configs[2]): ResNet-18 with per-EST BatchNorm, 16 ESTs x 32 CIFAR-shaped images
    (paper_2208_14228_b200/resnet.py).  Throughput with all 16 ESTs on this GPU (CUDA events); the C3
    schedule itself -- 2 steps on 8 launch groups ("GPUs"), rescale to 4, 2 steps, rescale to 2, 2 steps,
    per-EST BN statistics and cursors moved by the slot-copy kernel -- checked bit-identical against
    the uninterrupted run, with the context-switch time of each rescale."""
    from paper_2208_14228_b200.resnet import ResNetJob

    job = ResNetJob(ests=ests, batch=batch, gpus=1)
    s = torch.cuda.current_stream()
    for _ in range(warmup):
        job.step()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(s)
    for _ in range(steps):  # the non-finite check once after the timed steps (the update is guarded on device)
        losses = job.step(check=False)
    e1.record(s)
    e1.synchronize()
    job.check_status()
    ms = e0.elapsed_time(e1) / steps
    flops = job.flops_per_step()
    del job
    torch.cuda.empty_cache()
    from paper_2208_14228_b200.runlog import RunRecord, bitdiff

    a, b = ResNetJob(ests=ests, batch=batch, gpus=8), ResNetJob(ests=ests, batch=batch, gpus=1)
    for gpus in (4, 2):  # the planner knows the schedule: the layouts' buffers and step graphs are staged ahead
        a.prepare(gpus)
    switch_us, switch_host_us, first_ms = [], [], []
    la = None
    for gpus in (8, 4, 2):
        if gpus != 8:
            torch.cuda.synchronize()
            r0, r1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            t0 = time.perf_counter()
            r0.record(s)
            a.rescale(gpus)
            r1.record(s)
            t1 = time.perf_counter()
            r1.synchronize()
            switch_us.append(round(r0.elapsed_time(r1) * 1e3, 1))
            switch_host_us.append(round((t1 - t0) * 1e6, 1))
            pair = []
            for _ in range(2):  # the first step on the new layout (a replay of its staged graph), then the next
                f0, f1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                f0.record(s)
                lo = a.step()
                f1.record(s)
                f1.synchronize()
                pair.append(round(f0.elapsed_time(f1), 3))
                la.add(RunRecord(a.step_idx, [float(x) for x in lo.tolist()], a.fingerprint()))
            first_ms.append(pair)
        else:
            la = a.run_log(2, la)
    lb = b.run_log(6)
    sa, sb = a.est_state(), b.est_state()
    same = bool(torch.equal(a.params.view(torch.int32), b.params.view(torch.int32)) and
                torch.equal(sa["run_mean"].view(torch.int32), sb["run_mean"].view(torch.int32)) and
                torch.equal(sa["run_var"].view(torch.int32), sb["run_var"].view(torch.int32))) and bitdiff(la, lb) is None
    del a, b
    torch.cuda.empty_cache()
    return {"workload": "C3: ResNet-18 (CIFAR layout, widths 64-512) with per-EST BatchNorm, 16 ESTs x 32 "
                        "synthetic 32x32x3 images, softmax CE, momentum SGD (BASELINE.json configs[2])",
            "samples_per_s": round(ests * batch / (ms / 1e3), 1), "unit": "images/s", "ms_per_step": round(ms, 3),
            "conv_tflops_step_level": round(flops / ms / 1e9, 1), "loss": round(losses.mean().item(), 5),
            "rescale_8_4_2": {"schedule": "2 steps @8, rescale, 2 @4, rescale, 2 @2 vs 6 steps @1",
                              "bit_identical_weights_and_bn_stats": same, "context_switch_us": switch_us,
                              "context_switch_host_us": switch_host_us,
                              "first_and_second_step_after_switch_ms": first_ms,
                              "context_switch": "one bt_est_slot_copy launch (128-bit copies of every EST's BN "
                                                "statistics and cursor into its new owner's slots); the new "
                                                "layout's buffers and step graph staged ahead (ResNetJob.prepare)",
                              "run_logs": "per-EST losses + weight fingerprint per step, runlog.bitdiff: no divergence",
                              "weights_fp": la.records[-1].param_hash}}


def _oracle_run(threads: int):
    sys.path.insert(0, str(ROOT / "oracle"))
    import oracle

    run = oracle.Run(seed=SEED, max_workers=E_TOTAL, micro_batch=MICRO, dataset_size=NROWS, mode="d1",
                     layout=("gpu_fast",))
    run.set_threads(threads)
    return run


def oracle_threads() -> int:
    """The host-thread count the CPU port runs fastest with: the 8 ESTs of a mini-batch fan out over
    persistent spinning workers (bit-identical results); the serial allreduce + SGD bounds the gain.
    Calibrated on a short sample of each candidate up to the host's cores."""
    sys.path.insert(0, str(ROOT / "oracle"))
    import oracle

    cores = oracle.host_cores()
    best, best_t = 1, None
    for th in (1, 2, 4, 8):
        if th > max(1, cores - 1) or th > E_TOTAL:
            break
        run = _oracle_run(th)
        run.steps(200)
        t0 = time.perf_counter()
        run.steps(2000)
        el = time.perf_counter() - t0
        del run
        if best_t is None or el < best_t:
            best, best_t = th, el
    return best


def cpu_baseline(seconds: float, threads: int = 1):
    """The CPU oracle (C restatement of the reference) on the same C2 workload, bounded in time."""
    run = _oracle_run(threads)
    steps = 0
    t0 = time.perf_counter()
    while True:
        run.steps(1024)
        steps += 1024
        el = time.perf_counter() - t0
        if el >= seconds:
            break
    return steps * SAMPLES_PER_STEP / el, steps, el, run


def reference_arm(args, rank: int):
    """--impl reference: the reference's CPU implementation of the path (the C oracle port; the
    reference itself is Python and does not compile), on the host cores, same config/metric."""
    if rank != 0:
        return
    sys.path.insert(0, str(ROOT / "oracle"))
    import oracle

    cores = oracle.host_cores()
    threads = oracle_threads()
    run = _oracle_run(threads)
    run.steps(args.warmup)
    t0 = time.perf_counter()
    run.steps(args.steps)
    el = time.perf_counter() - t0
    v = args.steps * SAMPLES_PER_STEP / el
    line = {"impl": "reference", "metric": METRIC, "value": round(v, 1), "unit": "samples/s", "n_gpus": args.gpus,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": el * 1e3 / args.steps,
            "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": config_block(args.gpus),
            "cpu_baseline": {"value": round(v, 1), "unit": "samples/s", "cores": threads, "kind": "port",
                             "sample": f"{args.steps} C2 mini-batches after {args.warmup} warm-up, {threads} threads "
                                       f"(calibrated fastest of 1/2/4/8) of {cores} host cores"},
            "e2e": {"value": round(v, 1), "unit": "samples/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line))


def config_block(n):
    return {"workload": "C2: reference MLP (8-16-1 tanh, dropout 0.5, MSE), 8 ESTs x micro-batch 4, seed 42, "
                        "1024-row synthetic dataset, d1 / Tree(2) kind, momentum SGD (BASELINE.json configs[1])",
            "ests": E_TOTAL, "micro_batch": MICRO, "global_batch": SAMPLES_PER_STEP, "dataset_rows": NROWS,
            "parallelism": f"est-dp{n}", "l2": "flushed (256 MiB write) between timed launches; " + (
                f"each launch = {LAUNCH} mini-batches" if n == 1 else "each timed span = one epoch of 32 mini-batches")}


# Critical-path (latency) floor of one C2 mini-batch in the fused step kernel: the dependent
# chain every mini-batch must traverse, priced with latencies measured on the B200
# (tools/ubench*.cu), in SM cycles.
LATENCY_FLOOR_CYCLES = {
    "pre-activation chain (1 DMUL + 8 dependent DADD)": 72,
    "glibc tanh (branch-free form)": 550,
    "hidden -> shared -> warp (store, syncwarp, load)": 60,
    "output fold (16 dependent DADD) + error + gy": 152,
    "dz (3 DMUL + DSUB) + CTA barrier": 82,
    "gradient fold (loads + DMUL + 2-level tree)": 54,
    "one DSMEM slot exchange hop (st.async + mbarrier)": 500,
    "allreduce fold (loads + 3-level tree) + /E": 62,
    "momentum SGD (2 DMUL + DADD + DSUB) + commit barrier": 82,
}


def latency_floor(us_per_step: float, sm_mhz: float | None) -> dict:
    cyc = sum(LATENCY_FLOOR_CYCLES.values())
    mhz = sm_mhz or 1965.0
    floor_us = cyc / mhz
    return {"bound": "latency", "floor_us_per_step": round(floor_us, 3), "achieved_us_per_step": round(us_per_step, 3),
            "frac": round(floor_us / us_per_step, 4), "floor_cycles": cyc, "sm_mhz": mhz,
            "chain": LATENCY_FLOOR_CYCLES}


def _spawn_ranks(n: int) -> int:
    """`--gpus N` without a launcher: re-run this command under torch.distributed.run with N
    local ranks (127.0.0.1 rendezvous); rank 0 prints the line."""
    import socket

    sock = socket.socket()
    sock.bind(("127.0.0.1", 0))
    port = sock.getsockname()[1]
    sock.close()
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={n}",
           "--master-addr", "127.0.0.1", f"--master-port={port}", str(Path(__file__).resolve()), *sys.argv[1:]]
    return subprocess.run(cmd).returncode


def _rank_device(local: int) -> tuple[int, bool]:
    """(device index, shared): ranks beyond the visible GPU count share devices (tests on one GPU)."""
    n = torch.cuda.device_count()
    return local % n, n < int(os.environ.get("LOCAL_WORLD_SIZE", os.environ.get("WORLD_SIZE", "1")))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=3200)
    ap.add_argument("--warmup", type=int, default=64)
    ap.add_argument("--impl", default="b200", choices=["b200", "reference"])
    ap.add_argument("--cpu-seconds", type=float, default=10.0)
    ap.add_argument("--no-reducer", action="store_true")
    ap.add_argument("--no-bert", action="store_true", help="skip the C3 ResNet-18 and C4 BERT-base step measurements")
    ap.add_argument("--exchange", default="xdev", choices=["xdev", "ipc", "allgather"],
                    help="N>1: the lock-step persistent kernel over CUDA IPC peer memory (xdev), the per-step "
                         "peer-memory reducer (ipc), or an NCCL all-gather of EST slots")
    args = ap.parse_args()
    if args.warmup < 3:
        ap.error("--warmup must be >= 3")
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        sys.exit(_spawn_ranks(args.gpus))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if args.impl == "reference":
        return reference_arm(args, rank)

    import paper_2208_14228_b200 as bt

    devidx, shared = _rank_device(local)
    torch.cuda.set_device(devidx)
    dist = None
    hdev = "cuda"
    if world > 1:
        import torch.distributed as dist

        if shared:  # several ranks on one GPU (tests): NCCL refuses duplicate GPUs, gloo carries the host values
            dist.init_process_group("gloo")
            hdev = "cpu"
        else:
            dist.init_process_group("nccl", device_id=torch.device("cuda", devidx))
    peaks, peak_src = load_peaks()
    clocks = ClockSampler(devidx)
    flush_buf = torch.zeros(64 * 2**20, dtype=torch.float32, device="cuda")
    fl_n = [0]
    native_flush = os.environ.get("BT_FLUSH_NATIVE", "1") != "0"

    def flush():  # 256 MiB written (> the 126 MB L2) between timed launches
        if native_flush:
            fl_n[0] += 1
            _native_lib().bt_l2_flush(flush_buf.data_ptr(), flush_buf.numel() * 4, fl_n[0],
                                      torch.cuda.current_stream().cuda_stream)
        else:
            flush_buf.add_(1)

    rmb = None
    if world == 1:
        ts, ms, spans, launches, epc = bench_device_single(bt, args.steps, args.warmup, flush)
        final = np.array(ts.executors[0].model.values.tolist())
        ts_e, ms_e2e, launches_e, h2d, d2h, _ = bench_e2e_single(bt, args.steps, args.warmup, flush)
        final_e = np.array(ts_e.executors[0].model.values.tolist())
        assert np.array_equal(final.view(np.uint64), final_e.view(np.uint64)), "e2e and device runs diverged"
        rmb = bench_run_minibatch(bt)
        exchange = None
    else:
        exchange = args.exchange
        try:
            params, ms, launches, _, _ = bench_device_dist(bt, args.steps, args.warmup, rank, world, flush, False,
                                                           exchange)
        except Exception as exc:  # e.g. no peer access between these GPUs: the NCCL all-gather path
            print(f"bench: exchange={exchange} failed ({exc}); using allgather", file=sys.stderr)
            exchange = "allgather"
            params, ms, launches, _, _ = bench_device_dist(bt, args.steps, args.warmup, rank, world, flush, False,
                                                           exchange)
        final = params.cpu().numpy()
        params_e, ms_e2e, launches_e, h2d, d2h = bench_device_dist(bt, args.steps, args.warmup, rank, world, flush,
                                                                   True, exchange)
        epc = E_TOTAL // world
    if world > 1:
        t = torch.tensor([ms, ms_e2e], dtype=torch.float64, device=hdev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms, ms_e2e = t.tolist()
    weights_fnv = f"{bt.fnv1a64(final.astype('<f8').tobytes()):016x}"
    if world > 1:
        same, _ = replicas_identical(dist, final.astype("<f8").tobytes())
        assert same, "ranks hold different weights"

    value = args.steps * SAMPLES_PER_STEP / (ms / 1e3)
    e2e = args.steps * SAMPLES_PER_STEP / (ms_e2e / 1e3)
    reducer = None
    gemm = None
    bert = None
    reducer_dist = None
    if not args.no_reducer and world > 1 and (not shared or os.environ.get("BT_BENCH_C5_SHARED") == "1"):
        try:  # C5 across the GPUs of this run (NVLink); skipped when ranks share a GPU (no NVLink there)
            reducer_dist = bench_reducer_dist(rank, world, dist, peaks)
        except Exception as exc:
            reducer_dist = {"error": f"{type(exc).__name__}: {exc}"[:300]}
    if not args.no_reducer and rank == 0:
        reducer = bench_reducer(flush, peaks)
        gemm = bench_gemm(flush, peaks)
    resnet = None
    if not args.no_bert and world == 1:
        bert = bench_bert(peaks)
        resnet = bench_resnet(peaks)
    elif not args.no_bert:
        try:
            bert = bench_bert_dist(rank, world, dist)
        except Exception as exc:  # keep the headline line if the model-stack leg fails on this box
            bert = {"error": f"{type(exc).__name__}: {exc}"[:300]}
        try:
            resnet = bench_resnet_dist(rank, world, dist)
        except Exception as exc:
            resnet = {"error": f"{type(exc).__name__}: {exc}"[:300]}
    clk = clocks.stop()

    # Roofline of the step kernel: algorithmic HBM bytes per mini-batch = the 32 rows read
    # (32 x 9 x 8 B) + 8 losses written (64 B); per launch x steps in the launch.
    alg_step = SAMPLES_PER_STEP * 9 * 8 + E_TOTAL * 8
    per_launch_ms = ms / launches
    steps_per_launch = args.steps / launches
    achieved = alg_step * steps_per_launch / (per_launch_ms / 1e3) / 1e9
    us_step = ms * 1e3 / args.steps
    line = {
        "metric": METRIC, "value": round(value, 1), "unit": "samples/s", "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": ms / args.steps, "higher_is_better": True, "scaling": "strong",
        "vs_baseline": None, "dtype": "f64", "data": "synthetic (reference generator, seed 42)",
        "config": config_block(world),
        "e2e": {"value": round(e2e, 1), "unit": "samples/s", "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": d2h,
                "timing": "host clock around engine.run_steps (epoch lists recomputed on the host and copied "
                          "H2D, losses + status copied D2H, stream synchronised, all inside the span)"
                          if world == 1 else "CUDA events around the distributed steps"},
        "gpu_launches": launches,
        "roofline": {"kernel": "mlp_step_spec_kernel<8,8,2> (bt_mlp.cu: E=8, 8-CTA cluster, Tree(2))", "bound": "hbm", "achieved": round(achieved, 3),
                     "peak": peaks["hbm_gbs"], "unit": "GB/s", "frac": round(achieved / peaks["hbm_gbs"], 6),
                     "traffic": ncu_traffic("mlp_step_kernel"), "peak_source": peak_src,
                     "note": "latency-bound: one mini-batch is a ~1 kflop/sample dependent fp64 chain over 32 "
                             "samples; HBM and tensor rooflines do not bind -- see `latency` (DESIGN.md section 3.1)",
                     "us_per_step": round(us_step, 3), "est_per_cta": epc,
                     "latency": latency_floor(us_step, clk.get("sm_mhz"))},
        "weights_fnv": weights_fnv,  # FNV-1a of the final weights: equal for every N (bit-identical mappings)
        "clocks": clk,
    }
    if rmb is not None:
        line["run_minibatch"] = rmb
    if exchange is not None:
        line["config"]["exchange"] = exchange
    if reducer is not None:
        line["reducer"] = reducer
    if reducer_dist is not None:
        line["reducer_nvlink"] = reducer_dist
    if gemm is not None:
        line["gemm"] = gemm
    if bert is not None:
        line["c4_bert"] = bert
    if resnet is not None:
        line["c3_resnet"] = resnet
    if rank == 0 and world == 1 and args.cpu_seconds > 0:
        threads = oracle_threads()
        v, steps, el, run = cpu_baseline(args.cpu_seconds, threads)
        sys.path.insert(0, str(ROOT / "oracle"))
        import oracle

        line["cpu_baseline"] = {"value": round(v, 1), "unit": "samples/s", "cores": threads, "kind": "port",
                                "sample": f"{steps} C2 mini-batches ({el:.1f} s) of the C oracle, {threads} threads "
                                          f"(calibrated fastest of 1/2/4/8), {oracle.host_cores()} host cores present"}
    if rank == 0:
        print(json.dumps(line))
    if dist is not None:
        dist.barrier()
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
