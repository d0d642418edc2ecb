"""Per-EST FFN step (C4 slice) at BERT-base size: time per step, sequences/s, GEMM TF/s.

    python tools/ffn_bench.py [ests] [groups]
"""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import torch  # noqa: E402

from paper_2208_14228_b200.ffn import FFNJob  # noqa: E402

E = int(sys.argv[1]) if len(sys.argv) > 1 else 32
G = int(sys.argv[2]) if len(sys.argv) > 2 else 1
job = FFNJob(ests=E, tokens=1024)  # 8 sequences x 128 tokens per EST, d_model 768, d_ff 3072
groups = [E // G] * G
for _ in range(3):
    job.step(groups)
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
K = 10
e0.record()
for _ in range(K):
    losses = job.step(groups)
e1.record()
e1.synchronize()
ms = e0.elapsed_time(e1) / K
print(f"E={E} groups={groups}: {ms:.3f} ms/step, {E * 8 / ms * 1e3:.0f} sequences/s, "
      f"{job.flops_per_step() / ms / 1e9:.0f} TF/s (GEMM flops / step time), loss {losses.mean().item():.5f}")
