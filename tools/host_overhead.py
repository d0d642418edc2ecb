"""Host-side cost of the C2 launch path: ctypes, a plain launch, the cluster step launch, and a CUDA
graph replay of the same launch (device span of the replay beside it)."""

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


def host_us(fn, n=200):
    ts = []
    for _ in range(n):
        t0 = time.perf_counter()
        fn()
        ts.append((time.perf_counter() - t0) * 1e6)
    torch.cuda.synchronize()
    return round(statistics.median(ts[20:]), 2)


def main():
    L = _native.lib()
    cfg = bench.make_cfg(bt)
    ts = bt.init_training(cfg, [bt.ExecutorSpec("gpu_fast")])
    engine.run_steps(ts, 64)
    flags = torch.zeros(4, dtype=torch.int32, device="cuda")
    out = {"ctypes_noop_us": host_us(lambda: L.bt_abi_version()),
           "plain_launch_us": host_us(lambda: L.bt_flags_reset(flags.data_ptr(), stream()))}
    for K in (1, 20):
        losses = torch.empty((K, 8), dtype=torch.float64, device="cuda")
        a, keep = engine._step_args(ts, K, 4, None, losses, None)
        out[f"step_K{K}_launch_us"] = host_us(lambda: L.bt_mlp_step(C.byref(a), stream()), 100)
        g = torch.cuda.CUDAGraph()
        s = torch.cuda.Stream()
        s.wait_stream(torch.cuda.current_stream())
        with torch.cuda.stream(s):
            with torch.cuda.graph(g, stream=s):
                _native.check(L.bt_mlp_step(C.byref(a), stream()))
        torch.cuda.synchronize()
        out[f"graph_K{K}_replay_host_us"] = host_us(g.replay, 100)
        spans = []
        cs = torch.cuda.current_stream()
        for _ in range(30):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(cs)
            g.replay()
            e1.record(cs)
            e1.synchronize()
            spans.append(e0.elapsed_time(e1) * 1e3)
        out[f"graph_K{K}_span_us"] = round(statistics.median(spans[5:]), 2)
        spans = []
        for _ in range(30):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(cs)
            L.bt_mlp_step(C.byref(a), stream())
            e1.record(cs)
            e1.synchronize()
            spans.append(e0.elapsed_time(e1) * 1e3)
        out[f"eager_K{K}_span_us"] = round(statistics.median(spans[5:]), 2)
        # device-only: queue behind a busy kernel so the host launch cost is hidden
        busy = torch.empty(2**26, device="cuda")
        spans = []
        for _ in range(30):
            busy.add_(1)
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(cs)
            L.bt_mlp_step(C.byref(a), stream())
            e1.record(cs)
            e1.synchronize()
            spans.append(e0.elapsed_time(e1) * 1e3)
        out[f"queued_K{K}_span_us"] = round(statistics.median(spans[5:]), 2)
    print(json.dumps(out, indent=1))


if __name__ == "__main__":
    main()
