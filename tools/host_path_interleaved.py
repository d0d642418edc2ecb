"""Host-time split of a 20-mini-batch run_steps, the variants interleaved per iteration (so clock or
power drift hits all alike): the bare bt_mlp_run C-ABI call, _FastStep.run + bookkeeping, the whole
engine.run_steps -- resident lists -- and run_steps from host inputs (lists dropped: the sampled call).
Medians of 300 (microseconds)."""
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
engine.run_steps(ts, 20)
fs = engine._fast(ts)
L = _native.lib()
spe = ts.pipeline.steps_per_epoch
K = 20


def resident():
    gs = ts.global_step
    ts.pipeline.device_lists(gs // spe, (gs + K - 1) // spe)


def bare():
    L.bt_mlp_run(C.byref(fs.a), fs.host_io_ptr + 8 * (fs.KMAX - K) * fs.E, None,
                 torch.cuda.current_stream().cuda_stream)


def fast():
    ts.pipeline.advance_range(ts.global_step, K)
    fs.run(ts, K)
    engine._finish_steps(ts, K)


def whole():
    engine.run_steps(ts, K)


def sampled():
    ts.pipeline.drop_lists()
    engine.run_steps(ts, K)


acc = {k: [] for k in ("bare", "fast", "whole", "sampled")}
for it in range(320):
    for name, fn in (("bare", bare), ("fast", fast), ("whole", whole), ("sampled", sampled)):
        if name != "sampled":
            resident()
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        fn()
        acc[name].append((time.perf_counter() - t0) * 1e6)
print(json.dumps({k: round(statistics.median(v[20:]), 1) for k, v in acc.items()}))
