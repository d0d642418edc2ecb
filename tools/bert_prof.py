"""Kernel-time breakdown of one per-EST BERT step (torch.profiler / CUPTI), grouped by kernel name
(BT_PROF_RAW=1: every kernel name on its own line).

    python tools/bert_prof.py [ests] [layers] [seqs]
"""
import os
import sys
from collections import defaultdict
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import torch  # noqa: E402
from torch.profiler import ProfilerActivity, profile  # noqa: E402

from paper_2208_14228_b200.bert import BertJob  # noqa: E402

E = int(sys.argv[1]) if len(sys.argv) > 1 else 32
NL = int(sys.argv[2]) if len(sys.argv) > 2 else 12
S = int(sys.argv[3]) if len(sys.argv) > 3 else 8
job = BertJob(ests=E, seqs=S, layers=NL, est_group=4 if E % 4 == 0 else 1, fanin=2)
for _ in range(2):
    job.step()
torch.cuda.synchronize()
NS = int(os.environ.get("BT_PROF_STEPS", "1"))  # steps profiled (per-step averages printed)
with profile(activities=[ProfilerActivity.CUDA]) as prof:
    for _ in range(NS):
        job.step()
    torch.cuda.synchronize()
tot = defaultdict(float)
cnt = defaultdict(int)
for ev in prof.events():
    if ev.device_type == torch.autograd.DeviceType.CUDA:
        name = ev.name
        for key in () if os.environ.get("BT_PROF_RAW") else ("gemm_bf16_tn_pair_kernel", "gemm_bf16_tn_kernel", "attn_fwd", "attn_bwd", "ln_fwd", "ln_bwd",
                    "transpose_kernel", "colsum", "reduce", "cast_t", "ln_fold", "mse", "data_kernel", "tokens_kernel",
                    "embed_fwd", "gather_rows", "scatter_rows", "ce_kernel", "ce_fold", "sort_segments",
                    "embed_grad", "pos_grad"):
            if key in name:
                name = key
                break
        tot[name] += (ev.device_time_total if hasattr(ev, "device_time_total") else ev.cuda_time_total) / NS
        cnt[name] += 1
all_us = sum(tot.values())
for k, v in sorted(tot.items(), key=lambda kv: -kv[1]):
    print(f"{v / 1e3:9.3f} ms  {100 * v / all_us:5.1f}%  x{cnt[k] // NS:4d}  {k[:90]}")
print(f"total kernel time {all_us / 1e3:.3f} ms")
