"""Why a 20-mini-batch run_steps from host inputs costs more after the bench's L2 flush than back to back:
host-clock medians (microseconds) of the same call after (a) nothing, (b) the 256 MiB flush + sync,
(c) the flush + sync + an empty-ish device op + sync (re-warms the launch path), (d) the flush + sync +
a 200 us host spin (core awake, caches warm), plus the device span (CUDA events) of the call after (b)."""
import json
import statistics
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch  # noqa: E402

import bench  # noqa: E402
import paper_2208_14228_b200 as bt  # noqa: E402
from paper_2208_14228_b200 import _native, engine  # noqa: E402

cfg = bench.make_cfg(bt)
ts = bt.init_training(cfg, [bt.ExecutorSpec("gpu_fast")])
engine.run_steps(ts, 20)
flush_buf = torch.empty(64 << 20, dtype=torch.int32, device="cuda")
L = _native.lib()
n = [0]
s = torch.cuda.current_stream()
tiny = torch.zeros(1, device="cuda")


def flush():
    n[0] += 1
    L.bt_l2_flush(flush_buf.data_ptr(), flush_buf.numel() * 4, n[0], s.cuda_stream)


def call():
    ts.pipeline.drop_lists()
    t0 = time.perf_counter()
    engine.run_steps(ts, 20)
    return (time.perf_counter() - t0) * 1e6


def prep_none():
    torch.cuda.synchronize()


def prep_flush():
    flush()
    torch.cuda.synchronize()


def prep_flush_warm():
    flush()
    tiny.add_(1)
    torch.cuda.synchronize()


def prep_flush_spin():
    flush()
    torch.cuda.synchronize()
    t = time.perf_counter()
    while time.perf_counter() - t < 200e-6:
        pass


out = {}
for name, prep in (("back_to_back", prep_none), ("after_flush", prep_flush), ("after_flush_then_tiny_op", prep_flush_warm),
                   ("after_flush_then_200us_spin", prep_flush_spin)):
    v = []
    for _ in range(60):
        prep()
        v.append(call())
    out[name] = round(statistics.median(v[5:]), 1)
sp = []
for _ in range(40):
    prep_flush()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    ts.pipeline.drop_lists()
    engine.run_steps(ts, 20)
    e1.record()
    e1.synchronize()
    sp.append(e0.elapsed_time(e1) * 1e3)
out["device_span_after_flush"] = round(statistics.median(sp[5:]), 1)
print(json.dumps(out))
