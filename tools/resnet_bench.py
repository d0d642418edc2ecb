"""Per-EST ResNet-18 step with BatchNorm (C3): 16 ESTs x 32 images, images/s, and the cost of an
elastic rescale (EST context switch of the per-EST slots).

    python tools/resnet_bench.py [ests] [batch] [gpus]
"""
import os
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import torch  # noqa: E402

from paper_2208_14228_b200.resnet import ResNetJob  # noqa: E402

E = int(sys.argv[1]) if len(sys.argv) > 1 else 16
B = int(sys.argv[2]) if len(sys.argv) > 2 else 32
G = int(sys.argv[3]) if len(sys.argv) > 3 else 1
W, K = int(os.environ.get("BT_BENCH_WARMUP", "3")), int(os.environ.get("BT_BENCH_STEPS", "10"))
job = ResNetJob(ests=E, batch=B, gpus=G)
for _ in range(W):
    job.step()
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(K):
    losses = job.step()
e1.record()
e1.synchronize()
ms = e0.elapsed_time(e1) / K
r0, r1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
r0.record()
job.rescale(max(1, G // 2) if G > 1 else 2)
r1.record()
r1.synchronize()
print(f"ResNet-18 E={E} B={B} gpus={G}: {ms:.2f} ms/step, {E * B / ms * 1e3:.0f} images/s, "
      f"{job.flops_per_step() / ms / 1e9:.0f} TF/s conv, loss {losses.mean().item():.4f}, "
      f"rescale {r0.elapsed_time(r1) * 1e3:.0f} us, mem {torch.cuda.max_memory_allocated() / 2**30:.1f} GiB")
