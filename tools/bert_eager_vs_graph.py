"""Step time of the per-rank C4 work at N = 4 / 8 (8 or 4 ESTs on this GPU), eager launches vs the CUDA graph:
whether the multi-GPU legs (no graph across processes) are launch-bound."""
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import torch  # noqa: E402

from paper_2208_14228_b200.bert import BertJob  # noqa: E402

for E, graph, CHECK in ((8, True, True), (8, False, True), (8, False, False), (4, True, True), (4, False, True),
                        (4, False, False)):
    if True:
        job = BertJob(ests=E, est_group=4, fanin=2, graph=graph)
        for _ in range(3):
            job.step()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        t0 = time.perf_counter()
        e0.record()
        for _ in range(5):
            job.step(check=CHECK)
        e1.record()
        host = (time.perf_counter() - t0) / 5 * 1e3
        e1.synchronize()
        job.check_status()
        print(f"E={E} graph={graph} per-step check={CHECK}: {e0.elapsed_time(e1) / 5:.2f} ms/step "
              f"(host enqueue {host:.2f} ms/step)")
        del job
        torch.cuda.empty_cache()
