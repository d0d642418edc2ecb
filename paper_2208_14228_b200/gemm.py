"""Deterministic tensor-core GEMM (csrc/bt_gemm.cu) -- the dense-layer brick of
the C3/C4 model stack.

`gemm_bf16(a, b)` = a @ b.T for bf16 `a` [M, K] and `b` [N, K] (the nn.Linear
layout), fp32 accumulation on the tcgen05 tensor cores, fp32 or bf16 out.
One CTA owns each output tile and walks K in ascending order, so the result's
bits depend only on the inputs and the shape -- not on the grid size, the SM
count or the GPU: an EST's gradients do not change when it is remapped.
"""

from __future__ import annotations

import torch

from . import _native
from .device import require_cuda, stream
from .errors import InputError


def _out(out, shape, dtype, device):
    if out is None:
        return torch.empty(shape, dtype=dtype, device=device)
    if out.dtype != dtype or out.numel() != int(torch.Size(shape).numel()) or not out.is_contiguous():
        raise InputError(f"out must be a contiguous {dtype} tensor of {shape}")
    return out


def gemm_bf16(a: torch.Tensor, b: torch.Tensor, out_dtype: torch.dtype = torch.float32, grid: int = 0,
              out: torch.Tensor | None = None) -> torch.Tensor:
    require_cuda()
    if a.dtype != torch.bfloat16 or b.dtype != torch.bfloat16 or not (a.is_cuda and b.is_cuda):
        raise InputError("gemm_bf16 takes CUDA bfloat16 tensors")
    if a.dim() != 2 or b.dim() != 2 or a.shape[1] != b.shape[1]:
        raise InputError(f"gemm_bf16 shapes {tuple(a.shape)} x {tuple(b.shape)}^T")
    if out_dtype not in (torch.float32, torch.bfloat16):
        raise InputError("out_dtype must be float32 or bfloat16")
    a, b = a.contiguous(), b.contiguous()
    M, K = a.shape
    N = b.shape[0]
    c = _out(out, (M, N), out_dtype, a.device)
    _native.check(_native.lib().bt_gemm_bf16_tn(a.data_ptr(), b.data_ptr(), c.data_ptr(), M, N, K,
                                                 1 if out_dtype == torch.bfloat16 else 0, grid, stream()),
                  "gemm_bf16")
    return c


def gemm_bf16_batched(a: torch.Tensor, b: torch.Tensor, out_dtype: torch.dtype = torch.float32,
                      grid: int = 0, out: torch.Tensor | None = None) -> torch.Tensor:
    """c[e] = a[e] @ b[e].T for bf16 a [E, M, K], b [E, N, K] (one launch; per-entry bits equal the
    single-GEMM bits -- e.g. one weight gradient per EST, reduced afterwards in EST-rank order)."""
    require_cuda()
    if a.dtype != torch.bfloat16 or b.dtype != torch.bfloat16 or not (a.is_cuda and b.is_cuda):
        raise InputError("gemm_bf16_batched takes CUDA bfloat16 tensors")
    if a.dim() != 3 or b.dim() != 3 or a.shape[0] != b.shape[0] or a.shape[2] != b.shape[2]:
        raise InputError(f"gemm_bf16_batched shapes {tuple(a.shape)} x {tuple(b.shape)}^T")
    a, b = a.contiguous(), b.contiguous()
    E, M, K = a.shape
    N = b.shape[1]
    c = _out(out, (E, M, N), out_dtype, a.device)
    _native.check(_native.lib().bt_gemm_bf16_tn_batched(a.data_ptr(), b.data_ptr(), c.data_ptr(), E, M, N, K,
                                                         M * K, N * K, 1 if out_dtype == torch.bfloat16 else 0,
                                                         grid, stream()), "gemm_bf16_batched")
    return c


def gemm_bf16_at_b(a: torch.Tensor, b: torch.Tensor, out_dtype: torch.dtype = torch.float32, grid: int = 0,
                   out: torch.Tensor | None = None) -> torch.Tensor:
    """c[e] = a[e].T @ b[e] for bf16 a [E, K, M], b [E, K, N] (M, N contiguous: token-major
    activations): both operands are loaded MN-major by TMA, so e.g. a per-EST weight gradient
    dW_e = dY_e^T X_e needs no transposed copies.  Same determinism as gemm_bf16."""
    require_cuda()
    if a.dtype != torch.bfloat16 or b.dtype != torch.bfloat16 or not (a.is_cuda and b.is_cuda):
        raise InputError("gemm_bf16_at_b takes CUDA bfloat16 tensors")
    if a.dim() == 2:
        a, b = a.unsqueeze(0), b.unsqueeze(0)
    if a.dim() != 3 or b.dim() != 3 or a.shape[0] != b.shape[0] or a.shape[1] != b.shape[1]:
        raise InputError(f"gemm_bf16_at_b shapes {tuple(a.shape)}^T x {tuple(b.shape)}")
    a, b = a.contiguous(), b.contiguous()
    E, K, M = a.shape
    N = b.shape[2]
    c = _out(out, (E, M, N), out_dtype, a.device)
    _native.check(_native.lib().bt_gemm_bf16_ex(a.data_ptr(), b.data_ptr(), c.data_ptr(), E, M, N, K, K * M, K * N,
                                                 M * N, 1 if out_dtype == torch.bfloat16 else 0, None, 1, grid,
                                                 stream()), "gemm_bf16_at_b")
    return c
