"""A few 128-mini-batch launches of the C2 step kernel (for ncu source-level sampling of the step loop)."""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import torch  # noqa: E402

import bench  # noqa: E402
import paper_2208_14228_b200 as bt  # noqa: E402
from paper_2208_14228_b200 import engine  # noqa: E402

ts = bt.init_training(bench.make_cfg(bt), [bt.ExecutorSpec("gpu_fast")])
for _ in range(4):
    engine.run_steps(ts, 128)
torch.cuda.synchronize()
