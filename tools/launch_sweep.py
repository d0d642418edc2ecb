"""Fixed cost vs per-mini-batch cost of the C2 step launch (bt_mlp_step), on the GPU.

For K in a sweep: the device span of one K-mini-batch launch (CUDA events, L2 flushed before),
the host time of the ctypes call, and the run_minibatch wall time per call."""

import ctypes as C
import json
import statistics
import sys
import time
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import bench  # noqa: E402
import paper_2208_14228_b200 as bt  # noqa: E402
from paper_2208_14228_b200 import _native, engine  # noqa: E402
from paper_2208_14228_b200.device import stream  # noqa: E402


def main():
    flush_buf = torch.zeros(64 * 2**20, dtype=torch.float32, device="cuda")
    cfg = bench.make_cfg(bt)
    ts = bt.init_training(cfg, [bt.ExecutorSpec("gpu_fast")])
    engine.run_steps(ts, 64)
    s = torch.cuda.current_stream()
    out = {}
    for K in (1, 2, 5, 10, 20, 40, 100):
        for flush in (True, False):
            spans, host = [], []
            for it in range(12):
                for st in range(K):
                    ts.pipeline.advance_all(ts.global_step + st)
                losses = torch.empty((K, 8), dtype=torch.float64, device="cuda")
                a, keep = engine._step_args(ts, K, 4, None, losses, None)
                if flush:
                    flush_buf.add_(1)
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                e0.record(s)
                t0 = time.perf_counter()
                _native.check(_native.lib().bt_mlp_step(C.byref(a), stream()))
                host.append((time.perf_counter() - t0) * 1e6)
                e1.record(s)
                e1.synchronize()
                spans.append(e0.elapsed_time(e1) * 1e3)
                engine._finish_steps(ts, K)
                ts.dev.invalidate()
            sp = statistics.median(spans[2:])
            out[f"K{K}_{'flush' if flush else 'warm'}"] = {"span_us": round(sp, 2), "us_per_step": round(sp / K, 3),
                                                           "host_call_us": round(statistics.median(host[2:]), 2)}
    # the reference API's per-step call
    wall = []
    for _ in range(200):
        t0 = time.perf_counter()
        bt.run_minibatch(ts)
        wall.append((time.perf_counter() - t0) * 1e6)
    out["run_minibatch_us"] = round(statistics.median(wall[20:]), 2)
    print(json.dumps(out, indent=1))


if __name__ == "__main__":
    main()
