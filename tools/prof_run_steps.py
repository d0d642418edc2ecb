"""cProfile of the e2e leg's call: engine.run_steps(ts, 20) from host inputs (the epoch lists dropped before
every call, as bench.py's e2e leg does), 300 calls."""
import cProfile
import io
import pstats
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import torch  # noqa: E402

import bench  # noqa: E402
import paper_2208_14228_b200 as bt  # noqa: E402
from paper_2208_14228_b200 import engine  # noqa: E402

cfg = bench.make_cfg(bt)
ts = bt.init_training(cfg, [bt.ExecutorSpec("gpu_fast")])
engine.run_steps(ts, 20)


def loop(n=300):
    for _ in range(n):
        ts.pipeline.drop_lists()
        engine.run_steps(ts, 20)


loop(20)
torch.cuda.synchronize()
t0 = time.perf_counter()
loop()
print(f"{(time.perf_counter() - t0) / 300 * 1e6:.1f} us per run_steps(20) from host inputs")
pr = cProfile.Profile()
pr.enable()
loop()
pr.disable()
s = io.StringIO()
pstats.Stats(pr, stream=s).sort_stats("tottime").print_stats(22)
print(s.getvalue())
