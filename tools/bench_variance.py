"""Spread of the driver-shaped C2 measurement (one timed launch of K mini-batches after W warm-up
steps, L2 flushed before it): repeat bench.bench_device_single in one process."""

import json
import sys
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import bench  # noqa: E402
import paper_2208_14228_b200 as bt  # noqa: E402

K = int(sys.argv[1]) if len(sys.argv) > 1 else 20
W = int(sys.argv[2]) if len(sys.argv) > 2 else 5
flush_buf = torch.zeros(64 * 2**20, dtype=torch.float32, device="cuda")


def flush():
    flush_buf.add_(1)


out = []
for rep in range(10):
    ts, ms, spans, launches, epc = bench.bench_device_single(bt, K, W, flush)
    out.append(round(ms * 1e3 / K, 3))
print(json.dumps({"K": K, "W": W, "us_per_step": out}))
