"""Where the host-clock e2e time of a 20-mini-batch run_steps call goes (bench e2e leg)."""
import json
import statistics
import sys
import time
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import bench  # noqa: E402
import paper_2208_14228_b200 as bt  # noqa: E402
from paper_2208_14228_b200 import engine  # noqa: E402

K = int(sys.argv[1]) if len(sys.argv) > 1 else 20
cfg = bench.make_cfg(bt)
ts = bt.init_training(cfg, [bt.ExecutorSpec("gpu_fast")])
engine.run_steps(ts, 5)
pipe = ts.pipeline
out = {}


def med(fn, n=30):
    t = []
    for _ in range(n):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        fn()
        t.append((time.perf_counter() - t0) * 1e6)
    return round(statistics.median(t[3:]), 1)


def cold():
    pipe._lists_dev = None
    pipe._lists_host.clear()
    engine.run_steps(ts, K)


def warm_lists():
    engine.run_steps(ts, K)


out["run_steps_cold_lists_us"] = med(cold)
out["run_steps_cached_lists_us"] = med(warm_lists)
out["host_fisher_yates_1_epoch_us"] = med(lambda: (pipe._lists_host.clear(), pipe._lists_for_epoch(0)))
out["device_lists_upload_us"] = med(lambda: (setattr(pipe, "_lists_dev", None), pipe.device_lists(0, 0)))
fs = engine._fast(ts)
out["bt_mlp_run_us"] = med(lambda: (pipe.advance_range(ts.global_step, K), fs.run(ts, K), engine._finish_steps(ts, K)))
print(json.dumps(out))

import ctypes as C  # noqa: E402

from paper_2208_14228_b200 import _native  # noqa: E402

a = fs.a
a.K = K
a.losses = fs.io_ptr + 8 * (fs.KMAX - K) * fs.E
L = _native.lib()
s = torch.cuda.current_stream()
res = {}
res["step_launch_then_sync_us"] = med(lambda: (L.bt_mlp_step(C.byref(a), s.cuda_stream), s.synchronize()))
res["bt_mlp_run_only_us"] = med(lambda: L.bt_mlp_run(C.byref(a), fs.host_io_ptr + 8 * (fs.KMAX - K) * fs.E, None,
                                                      s.cuda_stream))
res["empty_sync_us"] = med(lambda: s.synchronize())
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
sp = []
for _ in range(20):
    e0.record(s)
    L.bt_mlp_run(C.byref(a), fs.host_io_ptr + 8 * (fs.KMAX - K) * fs.E, None, s.cuda_stream)
    e1.record(s)
    e1.synchronize()
    sp.append(e0.elapsed_time(e1) * 1e3)
res["bt_mlp_run_device_span_us"] = round(statistics.median(sp[3:]), 1)
print(json.dumps(res))
