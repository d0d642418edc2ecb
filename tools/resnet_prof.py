"""Kernel-time breakdown of one per-EST ResNet-18 step (torch.profiler / CUPTI), grouped by kernel name.

    python tools/resnet_prof.py [ests] [batch] [gpus]
"""
import sys
from collections import defaultdict
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import torch  # noqa: E402
from torch.profiler import ProfilerActivity, profile  # noqa: E402

from paper_2208_14228_b200.resnet import ResNetJob  # noqa: E402

E = int(sys.argv[1]) if len(sys.argv) > 1 else 16
B = int(sys.argv[2]) if len(sys.argv) > 2 else 32
G = int(sys.argv[3]) if len(sys.argv) > 3 else 1
job = ResNetJob(ests=E, batch=B, gpus=G)
for _ in range(2):
    job.step()
torch.cuda.synchronize()
with profile(activities=[ProfilerActivity.CUDA]) as prof:
    job.step()
    torch.cuda.synchronize()
tot, cnt = defaultdict(float), defaultdict(int)
for ev in prof.events():
    if ev.device_type == torch.autograd.DeviceType.CUDA:
        name = ev.name.split("(")[0][:80]
        tot[name] += ev.device_time_total
        cnt[name] += 1
all_us = sum(tot.values())
for k, v in sorted(tot.items(), key=lambda kv: -kv[1]):
    print(f"{v / 1e3:9.3f} ms  {100 * v / all_us:5.1f}%  x{cnt[k]:4d}  {k}")
print(f"total kernel time {all_us / 1e3:.3f} ms")
if "--seq" in sys.argv:
    evs = [ev for ev in prof.events() if ev.device_type == torch.autograd.DeviceType.CUDA]
    evs.sort(key=lambda e: e.time_range.start)
    for ev in evs:
        print(f"{ev.device_time_total:9.1f} us  {ev.name.split('(')[0][:90]}")
