"""Per-stage cycle breakdown of the fused step kernel (bt_mlp_step_profiled)."""
import ctypes as C
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import torch  # noqa: E402

import paper_2208_14228_b200 as bt  # noqa: E402
from paper_2208_14228_b200 import _native, engine  # noqa: E402
from paper_2208_14228_b200.device import stream  # noqa: E402

SHAPES = [tuple(int(v) for v in a.split(',')) for a in sys.argv[1:]] or [(8, 4, 32), (8, 4, 32), (16, 8, 32), (64, 4, 32)]
for shape in SHAPES:
    E, B, K = shape[:3]
    EPC = shape[3] if len(shape) > 3 else None
    cfg = bt.TrainRunConfig(seed=42, max_workers=E, micro_batch=B, dataset_size=max(1024, E * B * 32), lr=0.02,
                            momentum=0.9, dropout_rate=0.5, jitter=0.1, bucket_capacity=64,
                            determinism=bt.DeterminismMode.from_label("d1"), device_fanins={"gpu_fast": 2})
    ts = bt.init_training(cfg, [bt.ExecutorSpec("gpu_fast")])
    engine.run_steps(ts, 8)
    timing = torch.zeros(16, dtype=torch.int64, device="cuda")
    for st in range(K):
        ts.pipeline.advance_all(ts.global_step + st)
    losses = torch.empty((K, E), dtype=torch.float64, device="cuda")
    a, keep = engine._step_args(ts, K, B, None, losses, None)
    if EPC:
        a.est_per_cta = EPC
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    ev0.record()
    _native.check(_native.lib().bt_mlp_step_profiled(C.byref(a), timing.data_ptr(), stream()))
    ev1.record()
    ev1.synchronize()
    t = timing.tolist()
    n = max(t[5], 1)
    names = ["B+C rows..dz", "E grads+push", "exchange wait", "F fold+sgd", "commit barrier"]
    per = [x / n for x in t[:5]]
    print(f"E={E} B={B} K={K} epc={a.est_per_cta}: launch {ev0.elapsed_time(ev1) * 1e3:.1f} us, "
          f"{sum(per):.0f} cyc/step: " + ", ".join(f"{nm} {v:.0f}" for nm, v in zip(names, per))
          + f" | prologue detail: init {t[6]}, params {t[7]}, idx {t[8]}, jitter {t[12]}, data wait {t[13]}, bar {t[14]}, cluster {t[15]}"
          + f" | prologue {t[9]} cyc, epilogue {t[10]} cyc, CTA total {t[11]} cyc = {t[11] / 1965:.2f} us @1965")
