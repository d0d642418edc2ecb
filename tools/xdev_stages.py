"""Per-stage cycles of the lock-step multi-device step (bt_mlp_step_profiled on every shard of an
engine job over n logical devices): where the exchange time goes."""

import ctypes as C
import sys
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import bench  # noqa: E402
import paper_2208_14228_b200 as bt  # noqa: E402
from paper_2208_14228_b200 import _native, engine  # noqa: E402

K = 100
for n in [int(x) for x in (sys.argv[1:] or ["2", "4", "8"])]:
    bt.set_devices([0] * n)
    ts = bt.init_training(bench.make_cfg(bt), [bt.ExecutorSpec("gpu_fast")] * n)
    bt.run_steps(ts, 10)
    xs = engine._xdev(ts)
    ts.pipeline.advance_range(ts.global_step, K)
    gs, spe = ts.global_step, ts.pipeline.steps_per_epoch
    lists, base = ts.pipeline.device_lists(gs // spe, (gs + K - 1) // spe)
    rot = engine._rot_tensor(ts)
    timings = [torch.zeros(16, dtype=torch.int64, device="cuda") for _ in ts.dev.shards]
    for a in xs.args:
        a.K, a.step0, a.lists, a.epoch_base, a.rot = K, gs, lists.data_ptr(), base, rot.data_ptr()
        a.lr, a.mu = 0.02, 0.9
    torch.cuda.synchronize()
    for a, sh, t in zip(xs.args, ts.dev.shards, timings):
        _native.check(_native.lib().bt_mlp_step_profiled(C.byref(a), t.data_ptr(), sh.stream.cuda_stream))
    torch.cuda.synchronize()
    names = ["B+C", "E+push (+remote stores)", "DSMEM wait", "F (+remote polls) fold+sgd", "commit"]
    for i, t in enumerate(timings):
        v = t.tolist()
        steps = max(v[5], 1)
        print(f"{n} devices, shard {i}: {sum(v[:5]) / steps:.0f} cyc/step: " +
              ", ".join(f"{nm} {x / steps:.0f}" for nm, x in zip(names, v[:5])))
bt.set_devices(None)
