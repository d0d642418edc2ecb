"""TFLOP/s of the deterministic tcgen05 GEMM vs cuBLAS (torch.matmul) on the same shapes.

    python tools/gemm_bench.py [M,N,K ...]
"""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import torch  # noqa: E402

from paper_2208_14228_b200.gemm import gemm_bf16  # noqa: E402

SHAPES = [tuple(int(v) for v in a.split(",")) for a in sys.argv[1:]] or [
    (8192, 8192, 8192), (4096, 4096, 4096), (32768, 768, 768), (32768, 3072, 768), (32768, 768, 3072)]
ITERS = 3 if len(sys.argv) > 1 else 20


def timeit(fn, iters=None):
    iters = iters or ITERS
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    best = 1e30
    for _ in range(3):
        e0.record()
        for _ in range(iters):
            fn()
        e1.record()
        e1.synchronize()
        best = min(best, e0.elapsed_time(e1) / iters)
    return best


for M, N, K in SHAPES:
    a = torch.randn(M, K, device="cuda").to(torch.bfloat16)
    b = torch.randn(N, K, device="cuda").to(torch.bfloat16)
    fl = 2.0 * M * N * K
    t_ours16 = timeit(lambda: gemm_bf16(a, b, torch.bfloat16))
    t_ours32 = timeit(lambda: gemm_bf16(a, b, torch.float32))
    t_cub = timeit(lambda: torch.matmul(a, b.T))
    print(f"{M}x{N}x{K}: ours bf16-out {fl / t_ours16 / 1e9:7.1f} TF/s ({t_ours16 * 1e3:8.1f} us), "
          f"f32-out {fl / t_ours32 / 1e9:7.1f} TF/s, cuBLAS bf16 {fl / t_cub / 1e9:7.1f} TF/s ({t_cub * 1e3:8.1f} us)")
