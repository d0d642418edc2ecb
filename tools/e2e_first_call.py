"""e2e leg diagnosis: host time of each run_steps call (after the flush, lists dropped) in sequence -- the first call at a new size vs repeats."""
import sys, time, json
sys.path.insert(0, str(__import__("pathlib").Path(__file__).resolve().parents[1]))
import torch, bench, paper_2208_14228_b200 as bt
from paper_2208_14228_b200 import engine, _native
cfg = bench.make_cfg(bt)
ts = bt.init_training(cfg, [bt.ExecutorSpec("gpu_fast")])
engine.run_steps(ts, 5)
torch.cuda.synchronize()
fb = torch.empty(64 << 20, dtype=torch.int32, device="cuda")
L = _native.lib(); s = torch.cuda.current_stream()
res = []
for i, n in enumerate([20, 20, 20, 7, 7, 20, 33, 33, 20]):
    L.bt_l2_flush(fb.data_ptr(), fb.numel() * 4, i + 1, s.cuda_stream)
    ts.pipeline._lists_dev = None; ts.pipeline._lists_host.clear()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    engine.run_steps(ts, n)
    res.append((n, round((time.perf_counter() - t0) * 1e6, 1)))
print(json.dumps(res))
