"""Inter-kernel gaps of one captured BERT step (torch.profiler): busy time, span, the largest gaps."""
import sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import torch
from torch.profiler import ProfilerActivity, profile
from paper_2208_14228_b200.bert import BertJob
job = BertJob(ests=32, est_group=4, fanin=2)
for _ in range(3):
    job.step()
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(5):
    job.step()
e1.record(); e1.synchronize()
print("step ms", e0.elapsed_time(e1) / 5)
with profile(activities=[ProfilerActivity.CUDA]) as prof:
    job.step()
    torch.cuda.synchronize()
evs = sorted([e for e in prof.events() if e.device_type == torch.autograd.DeviceType.CUDA], key=lambda e: e.time_range.start)
busy = sum(e.time_range.elapsed_us() for e in evs)
span = evs[-1].time_range.end - evs[0].time_range.start
gaps = [(evs[i + 1].time_range.start - evs[i].time_range.end, evs[i].name[:50], evs[i + 1].name[:50]) for i in range(len(evs) - 1)]
print("kernels", len(evs), "busy ms", busy / 1e3, "span ms", span / 1e3)
gs = sorted(gaps, key=lambda g: -g[0])
print("sum gaps ms", sum(max(0, g[0]) for g in gaps) / 1e3)
for g in gs[:15]:
    print(round(g[0], 1), "|", g[1], "->", g[2])
import collections
c = collections.Counter()
for g in gaps:
    if g[0] > 0: c[round(g[0])] += 1
print(sorted(c.items())[:20])
