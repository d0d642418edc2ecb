"""Host-time split of engine.run_steps(ts, 20) with resident lists: the whole call, _FastStep.run, and the
bare bt_mlp_run C-ABI call with the same argument block (medians of 200)."""
import ctypes as C
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


def med(fn, n=200):
    t = []
    for _ in range(n):
        t0 = time.perf_counter()
        fn()
        t.append((time.perf_counter() - t0) * 1e6)
    return round(statistics.median(t[20:]), 1)


spe = ts.pipeline.steps_per_epoch


def keep_resident():
    gs = ts.global_step
    ts.pipeline.device_lists(gs // spe, (gs + 19) // spe)


def whole():
    keep_resident()
    engine.run_steps(ts, 20)


def fast_only():
    keep_resident()
    ts.pipeline.advance_range(ts.global_step, 20)
    fs.run(ts, 20)
    engine._finish_steps(ts, 20)


def bare():
    L.bt_mlp_run(C.byref(fs.a), fs.host_io_ptr + 8 * (fs.KMAX - 20) * fs.E, None, torch.cuda.current_stream().cuda_stream)


print({"run_steps_us": med(whole), "fast_run_us": med(fast_only), "keep_resident_us": med(keep_resident),
       "bare_c_call_us": med(bare)})
