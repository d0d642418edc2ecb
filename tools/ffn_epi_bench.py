"""FFN GEMM epilogue cost at BERT-base shape: plain bf16 store vs bias+GELU (2 outputs) vs dropout'*GELU'."""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import torch  # noqa: E402

from paper_2208_14228_b200 import _native  # noqa: E402
from paper_2208_14228_b200.device import stream  # noqa: E402

T, D, F = 32768, 768, 3072
L = _native.lib()
a = torch.randn(T, D, device="cuda").to(torch.bfloat16)
w = torch.randn(F, D, device="cuda").to(torch.bfloat16)
c = torch.empty(T, F, device="cuda", dtype=torch.bfloat16)
c2 = torch.empty_like(c)
aux = torch.randn(T, F, device="cuda").to(torch.bfloat16)
bias = torch.zeros(F, device="cuda")


def timeit(fn, iters=20):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(iters):
        fn()
    e1.record()
    e1.synchronize()
    return e0.elapsed_time(e1) / iters * 1e3


fl = 2.0 * T * F * D
for name, fn in (
        ("plain bf16", lambda: L.bt_gemm_bf16_ex(a.data_ptr(), w.data_ptr(), c.data_ptr(), 1, T, F, D, 0, 0, 0, 1, None,
                                                 0, 0, stream())),
        ("bias bf16", lambda: L.bt_gemm_bf16_ex(a.data_ptr(), w.data_ptr(), c.data_ptr(), 1, T, F, D, 0, 0, 0, 1,
                                                bias.data_ptr(), 0, 0, stream())),
        ("ffn fwd (bias+gelu, 2 out)", lambda: L.bt_gemm_bf16_ffn(a.data_ptr(), w.data_ptr(), c.data_ptr(), T, F, D, 1,
                                                                   bias.data_ptr(), None, c2.data_ptr(), 1, 0, 0, 1024,
                                                                   0.0, 0, stream())),
        ("ffn bwd (gelu' of aux)", lambda: L.bt_gemm_bf16_ffn(a.data_ptr(), w.data_ptr(), c.data_ptr(), T, F, D, 2, None,
                                                               aux.data_ptr(), None, 1, 0, 0, 1024, 0.0, 0, stream()))):
    us = timeit(fn)
    print(f"{name:30s} {us:8.1f} us  {fl / us / 1e6:7.1f} TF/s")
