import sys; sys.path.insert(0, '/root/repo')
import torch
from paper_2208_14228_b200.gemm import gemm_bf16_at_b
def timeit(fn, iters=10):
    for _ in range(3): fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(iters): fn()
    e1.record(); e1.synchronize()
    return e0.elapsed_time(e1) / iters * 1e3
for B, K in ((8, 4096), (32, 1024)):
    tot = 0
    for M, N in ((768, 3072), (3072, 768), (768, 768), (2304, 768)):
        a = torch.randn(B, K, M, device="cuda").to(torch.bfloat16)
        b = torch.randn(B, K, N, device="cuda").to(torch.bfloat16)
        c = torch.empty(B, M, N, device="cuda")
        us = timeit(lambda: gemm_bf16_at_b(a, b, out=c))
        tot += us
        print(f"batch {B} K {K} M {M} N {N}: {us:7.1f} us  {2.0*B*K*M*N/us/1e6:7.1f} TF/s")
    print("sum", round(tot, 1), "us per layer")
