"""Per-statement host time of _FastStep.run's prologue (resident lists), medians of 300 (microseconds)."""
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
from paper_2208_14228_b200.device import ptr  # noqa: E402

cfg = bench.make_cfg(bt)
ts = bt.init_training(cfg, [bt.ExecutorSpec("gpu_fast")])
engine.run_steps(ts, 20)
fs = engine._fast(ts)
pipe = ts.pipeline
spe = pipe.steps_per_epoch
acc = {}


def tick(name, t0):
    t1 = time.perf_counter()
    acc.setdefault(name, []).append((t1 - t0) * 1e6)
    return t1


for _ in range(300):
    gs = ts.global_step
    pipe.device_lists(gs // spe, (gs + 19) // spe)
    t = time.perf_counter()
    pipe.advance_all(gs)
    t = tick("advance_all", t)
    f = engine._fast(ts)
    t = tick("_fast", t)
    rot = engine._rot_tensor(ts)
    t = tick("_rot_tensor", t)
    a = f.a
    a.K, a.step0 = 20, gs
    a.rot = ptr(rot)
    ex0 = ts.executors[0]
    a.lr, a.mu = float(ex0._lr), float(ex0._mu)
    a.losses = f.io_ptr + 8 * (f.KMAX - 20) * f.E
    t = tick("struct fields", t)
    ok = pipe.lists_resident(gs // spe, (gs + 19) // spe)
    lists, base = pipe.device_lists(gs // spe, (gs + 19) // spe)
    a.lists, a.epoch_base = lists.data_ptr(), base
    t = tick("lists", t)
    s = engine._raw_stream()
    t = tick("_raw_stream", t)
    st = _native.lib().bt_mlp_run(C.byref(a), f.host_io_ptr + 8 * (f.KMAX - 20) * f.E, None, s)
    t = tick("bt_mlp_run", t)
    f.dev.invalidate()
    out = f.rows_np[f.KMAX - 20:].copy()
    t = tick("after", t)
    pipe.advance_range(gs + 1, 19)
    engine._finish_steps(ts, 20)
    t = tick("advance_range+finish", t)
print({k: round(statistics.median(v[30:]), 2) for k, v in acc.items()})
