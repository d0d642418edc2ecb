"""Every GEMM/convolution launch of one C3 step in launch order with its duration (torch.profiler / CUPTI)."""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import torch  # noqa: E402
from torch.profiler import ProfilerActivity, profile  # noqa: E402

from paper_2208_14228_b200.resnet import ResNetJob  # noqa: E402

job = ResNetJob(ests=16, batch=32, gpus=1, graph=False)
for _ in range(2):
    job.step()
torch.cuda.synchronize()
with profile(activities=[ProfilerActivity.CUDA]) as prof:
    job.step()
    torch.cuda.synchronize()
evs = sorted([e for e in prof.events() if e.device_type == torch.autograd.DeviceType.CUDA], key=lambda e: e.time_range.start)
ALL = len(sys.argv) > 1 and sys.argv[1] == "all"  # every kernel, not only the GEMMs
for e in evs:
    if ALL or "gemm" in e.name or "conv" in e.name:
        print(f"{e.device_time_total:8.1f} us  {e.name[:100]}")
print("convs:", [(c.name, c.ci, c.co, c.k, c.s, c.hout) for c in job.convs])
