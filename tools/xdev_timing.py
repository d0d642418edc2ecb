"""Lock-step multi-device C2 step, timed: the engine over n logical devices (set_devices) running
launches of K mini-batches (host clock around run_steps, which synchronises), per mini-batch."""

import json
import sys
import time
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import bench  # noqa: E402
import paper_2208_14228_b200 as bt  # noqa: E402

devs = [int(x) for x in sys.argv[1].split(",")] if len(sys.argv) > 1 else [0]
out = {}
for n in (1, 2, 4, 8):
    bt.set_devices([devs[i % len(devs)] for i in range(n)])
    ts = bt.init_training(bench.make_cfg(bt), [bt.ExecutorSpec("gpu_fast")] * n)
    bt.run_steps(ts, 100)
    res = {}
    for K in (1, 20, 100):
        times = []
        for _ in range(10):
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            bt.run_steps(ts, K)
            times.append((time.perf_counter() - t0) * 1e6)
        times.sort()
        res[f"K{K}_us_per_step"] = round(times[len(times) // 2] / K, 3)
    out[f"{n}_devices"] = res
bt.set_devices(None)
print(json.dumps({"devices": devs, **out}))
