"""C5 sweep: the deterministic reducer (bt_reduce_update) over S = 1 MB..1 GB per EST, E = 8..64 ESTs.

Algorithmic HBM bytes per launch (G = 1) = E*S (gradient slots) + 4*S (param, velocity read+write).
Timed with CUDA events on the launching stream, median of `iters` launches, L2 flushed (256 MiB write)
between launches.  Prints one JSON document (profiles/<tag>_reducer_sweep.json).
"""
import ctypes as C
import json
import statistics
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import torch  # noqa: E402

from paper_2208_14228_b200 import _native  # noqa: E402
from paper_2208_14228_b200.device import Flags, stream  # noqa: E402

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
from bench import HostGate  # noqa: E402

PEAK = json.loads((Path(__file__).resolve().parent.parent / "MEASURED_PEAKS.json").read_text()).get("hbm_gbs", 6541.8) \
    if (Path(__file__).resolve().parent.parent / "MEASURED_PEAKS.json").exists() else 6541.8


def run(E, S_MB, fan, iters=7, dtype=torch.float32):
    es = torch.tensor([], dtype=dtype).element_size()
    n = S_MB * 2**20 // es
    g = torch.empty((E, n), dtype=dtype, device="cuda").uniform_(-1, 1)
    p = torch.empty(n, dtype=dtype, device="cuda").uniform_(-1, 1)
    v = torch.zeros(n, dtype=dtype, device="cuda")
    flags = Flags()
    flush = torch.empty(64 * 2**20, dtype=torch.float32, device="cuda")
    a = _native.ReduceArgs()
    a.dtype = _native.DTYPE_F32 if dtype == torch.float32 else _native.DTYPE_F64
    a.mode, a.E, a.fanin, a.n = _native.REDUCE_UPDATE, E, fan, n
    for k in range(E):
        a.grads[k] = g[k].data_ptr()
    a.param, a.vel, a.param_out, a.vel_out = p.data_ptr(), v.data_ptr(), p.data_ptr(), v.data_ptr()
    a.lr, a.mu, a.flags = 1e-9, 0.9, flags.t.data_ptr()
    _native.check(_native.lib().bt_reduce_update(C.byref(a), stream()))
    s = torch.cuda.current_stream()
    gate = HostGate()
    times = []
    for _ in range(iters):
        flush.add_(1)
        # the stream held at a device-side wait until [e0, launch, e1] are all queued: the span is the kernel
        # (bench.py's HostGate), not the host's launch latency
        gate.close(s)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        try:
            e0.record(s)
            _native.check(_native.lib().bt_reduce_update(C.byref(a), stream()))
            e1.record(s)
        finally:
            gate.open()
        e1.synchronize()
        times.append(e0.elapsed_time(e1))
    ms = statistics.median(times)
    alg = (E + 4) * n * es
    del g, p, v, flush
    torch.cuda.empty_cache()
    return {"E": E, "S_MB": S_MB, "variant": "sequential" if fan == 0 else f"tree{fan}", "dtype": str(dtype)[6:],
            "ms": round(ms, 4), "alg_bytes": alg, "gbs": round(alg / ms / 1e6, 1), "frac_hbm": round(alg / ms / 1e6 / PEAK, 4)}


if __name__ == "__main__":
    out = {"peak_hbm_gbs": PEAK, "peak_source": "MEASURED_PEAKS.json", "G": 1, "rows": []}
    for E in (8, 16, 32, 64):
        for S in (1, 4, 16, 64, 256, 1024):
            if E * S > 70 * 1024:
                continue
            for fan in (2, 0):
                r = run(E, S, fan)
                out["rows"].append(r)
                print(json.dumps(r), file=sys.stderr)
    print(json.dumps(out, indent=1))
