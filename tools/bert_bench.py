"""Per-EST BERT-base encoder step (C4): time per step, sequences/s, dense-GEMM TF/s.

    python tools/bert_bench.py [ests] [groups] [layers] [seqs]
"""
import os
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import torch  # noqa: E402

from paper_2208_14228_b200.bert import BertJob  # noqa: E402

E = int(sys.argv[1]) if len(sys.argv) > 1 else 32
G = int(sys.argv[2]) if len(sys.argv) > 2 else 1
NL = int(sys.argv[3]) if len(sys.argv) > 3 else 12
S = int(sys.argv[4]) if len(sys.argv) > 4 else 8
job = BertJob(ests=E, seqs=S, layers=NL, est_group=4 if E % 4 == 0 else 1, fanin=2)
groups = [E // G] * G
W, K = int(os.environ.get("BT_BENCH_WARMUP", "3")), int(os.environ.get("BT_BENCH_STEPS", "5"))
for _ in range(W):
    job.step(groups)
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(K):
    losses = job.step(groups)
e1.record()
e1.synchronize()
ms = e0.elapsed_time(e1) / K
print(f"BERT E={E} groups={groups} layers={NL} seqs/EST={S}: {ms:.2f} ms/step, {E * S / ms * 1e3:.0f} sequences/s, "
      f"{job.gemm_flops_per_step() / ms / 1e9:.0f} TF/s dense (+{job.attn_flops_per_step() / ms / 1e9:.0f} attn), "
      f"loss {losses.mean().item():.5f}, P={job.P}, mem {torch.cuda.max_memory_allocated() / 2**30:.1f} GiB")
