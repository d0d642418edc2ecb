"""Every GEMM launch of one C4 step in launch order with its duration (torch.profiler / CUPTI), labelled
by the BertJob call sequence, to see which dense products are below the tensor roofline."""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import torch  # noqa: E402
from torch.profiler import ProfilerActivity, profile  # noqa: E402

from paper_2208_14228_b200.bert import BertJob  # noqa: E402

NL = int(sys.argv[1]) if len(sys.argv) > 1 else 2
job = BertJob(ests=32, seqs=8, layers=NL, est_group=4, fanin=2, graph=False)
for _ in range(2):
    job.step()
torch.cuda.synchronize()
with profile(activities=[ProfilerActivity.CUDA]) as prof:
    job.step()
    torch.cuda.synchronize()
evs = [e for e in prof.events() if e.device_type == torch.autograd.DeviceType.CUDA]
evs.sort(key=lambda e: e.time_range.start)
T, D, F, V = 32768, 768, 3072, job.Vp
fwd = [("QKV", T, 3 * D, D), ("Wo", T, D, D), ("W1+GELU", T, F, D), ("W2", T, D, F)]
head = [("logits", 5120, V, D), ("dym", 5120, D, V), ("dWdec", V, D, 5120)]
bwd = [("dHpre(FFN bwd)", T, F, D), ("dX W1", T, D, F), ("dW W2", D, F, T), ("dW W1", F, D, T), ("dX Wo", T, D, D),
       ("dW Wo", D, D, T), ("dX QKV", T, D, 3 * D), ("dW QKV", 3 * D, D, T)]
labels = fwd * NL + head + bwd * NL
g = [e for e in evs if "gemm" in e.name]
print(f"{len(g)} GEMM launches, {len(labels)} labels")
tot = {}
for e, (name, M, N, K) in zip(g, labels):
    us = e.device_time_total
    tf = 2.0 * M * N * K / us / 1e6
    tot[name] = tot.get(name, 0) + us
    print(f"{name:16s} {M:6d}x{N:6d}x{K:6d} {us:8.1f} us {tf:7.1f} TF/s")
print({k: round(v, 1) for k, v in tot.items()})
