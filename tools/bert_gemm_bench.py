"""TF/s of each GEMM shape of the per-EST BERT-base step (T = 32 ESTs x 1024 tokens), ours vs cuBLAS.

    python tools/bert_gemm_bench.py
"""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import torch  # noqa: E402

from paper_2208_14228_b200 import _native  # noqa: E402
from paper_2208_14228_b200.device import stream  # noqa: E402

T, D, F, E, Te = 32768, 768, 3072, 32, 1024


def timeit(fn, iters=10):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(iters):
        fn()
    e1.record()
    e1.synchronize()
    return e0.elapsed_time(e1) / iters


def ours(M, N, K, batch=1, out_bf16=False):
    a = torch.randn(batch, M, K, device="cuda").to(torch.bfloat16)
    b = torch.randn(batch, N, K, device="cuda").to(torch.bfloat16)
    c = torch.empty(batch, M, N, device="cuda", dtype=torch.bfloat16 if out_bf16 else torch.float32)
    L = _native.lib()
    f = lambda: _native.check(L.bt_gemm_bf16_tn_ex(a.data_ptr(), b.data_ptr(), c.data_ptr(), batch, M, N, K, M * K,  # noqa: E731
                                                   N * K, M * N, 1 if out_bf16 else 0, None, 0, stream()))
    g = lambda: torch.bmm(a, b.transpose(1, 2)) if batch > 1 else torch.matmul(a[0], b[0].T)  # noqa: E731
    fl = 2.0 * batch * M * N * K
    t, tc = timeit(f), timeit(g)
    print(f"{batch:3d} x {M}x{N}x{K} {'bf16' if out_bf16 else 'f32 '}: ours {fl / t / 1e9:7.1f} TF/s ({t * 1e3:7.1f} us)"
          f"  cuBLAS(bf16 out) {fl / tc / 1e9:7.1f} TF/s ({tc * 1e3:7.1f} us)")
    return t


tot = 0
for M, N, K, bf in ((T, 3 * D, D, True), (T, D, D, False), (T, F, D, True), (T, D, F, False),
                    (T, F, D, True), (T, D, F, False), (T, D, D, True), (T, D, 3 * D, False)):
    tot += ours(M, N, K, out_bf16=bf)
for M, N in ((D, F), (F, D), (D, D), (3 * D, D)):
    tot += ours(M, N, Te, batch=E)
print(f"sum of one layer's GEMMs: {tot:.3f} ms -> x12 = {12 * tot:.2f} ms")
