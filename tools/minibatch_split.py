"""Where run_minibatch's time goes (the reference API's per-step call, K = 1): host-clock medians of 300,
the variants interleaved per iteration -- the whole call, _FastStep.run + bookkeeping, the bare bt_mlp_run
C-ABI call with the same argument block, and the device span of that call (CUDA events)."""
import ctypes as C
import json
import statistics
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import torch  # noqa: E402

import bench  # noqa: E402
import paper_2208_14228_b200 as bt  # noqa: E402
from paper_2208_14228_b200 import _native, engine  # noqa: E402

cfg = bench.make_cfg(bt)
ts = bt.init_training(cfg, [bt.ExecutorSpec("gpu_fast")])
for _ in range(30):
    bt.run_minibatch(ts)
fs = engine._fast(ts)
L = _native.lib()
s = torch.cuda.current_stream()


def whole():
    bt.run_minibatch(ts)


def fast():
    ts.pipeline.advance_all(ts.global_step)
    fs.run(ts, 1)
    engine._finish_steps(ts, 1)


def bare():
    L.bt_mlp_run(C.byref(fs.a), fs.host_io_ptr + 8 * (fs.KMAX - 1) * fs.E, None, s.cuda_stream)


def launch_only():
    L.bt_mlp_step(C.byref(fs.a), s.cuda_stream)


acc = {k: [] for k in ("run_minibatch", "fast", "bare_bt_mlp_run", "launch_call_only")}
for it in range(320):
    for name, fn in (("run_minibatch", whole), ("fast", fast), ("bare_bt_mlp_run", bare), ("launch_call_only", launch_only)):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        fn()
        acc[name].append((time.perf_counter() - t0) * 1e6)
torch.cuda.synchronize()
out = {k: round(statistics.median(v[20:]), 1) for k, v in acc.items()}
sp = []
for _ in range(50):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    e0.record()
    L.bt_mlp_step(C.byref(fs.a), s.cuda_stream)
    e1.record()
    e1.synchronize()
    sp.append(e0.elapsed_time(e1) * 1e3)
out["device_span_one_minibatch"] = round(statistics.median(sp[5:]), 1)
print(json.dumps(out))
