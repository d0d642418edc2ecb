"""Profiling driver: one long persistent launch of the C2 step (for ncu source-level sampling)."""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import torch  # noqa: E402

import paper_2208_14228_b200 as bt  # noqa: E402
from paper_2208_14228_b200 import engine  # noqa: E402

E = int(sys.argv[1]) if len(sys.argv) > 1 else 8
B = int(sys.argv[2]) if len(sys.argv) > 2 else 4
K = int(sys.argv[3]) if len(sys.argv) > 3 else 2000
cfg = bt.TrainRunConfig(seed=42, max_workers=E, micro_batch=B, dataset_size=1024 * max(1, E * B // 32), lr=0.02,
                        momentum=0.9, dropout_rate=0.5, jitter=0.1, bucket_capacity=64,
                        determinism=bt.DeterminismMode.from_label("d1"), device_fanins={"gpu_fast": 2})
ts = bt.init_training(cfg, [bt.ExecutorSpec("gpu_fast")])
engine.run_steps(ts, 64)
torch.cuda.synchronize()
s = torch.cuda.Event(enable_timing=True)
e = torch.cuda.Event(enable_timing=True)
s.record()
engine.run_steps(ts, K)
e.record()
e.synchronize()
print(f"E={E} B={B} K={K}: {s.elapsed_time(e) * 1e3 / K:.3f} us/step (one launch, incl. host bookkeeping)")
