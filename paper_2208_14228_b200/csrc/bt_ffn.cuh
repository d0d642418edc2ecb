// bt_ffn.cuh -- element math of the per-EST FFN step, shared by the fused
// GEMM epilogues (bt_gemm.cu) and the standalone kernels (bt_ffn.cu).
// All randomness is counter-form splitmix64 keyed by (seed, global EST rank,
// step, element) -- never by the launch, tile or GPU.
#pragma once

#include <cuda_bf16.h>
#include <stdint.h>

#include "bt_common.cuh"

namespace bt {
namespace ffn {

constexpr uint64_t TAG_FFN_X = 0x4646'4e5f'5844'4154ull;     // "FFN_XDAT"
constexpr uint64_t TAG_FFN_Y = 0x4646'4e5f'5944'4154ull;     // "FFN_YDAT"
constexpr uint64_t TAG_FFN_DROP = 0x4646'4e5f'4452'4f50ull;  // "FFN_DROP"

__device__ __forceinline__ float uniform_pm1(uint64_t stream, uint64_t n) {  // [-1, 1)
  return (float)(unit_float(draw_raw(stream, n)) * 2.0 - 1.0);
}

// Dropout masks: one splitmix64 draw per PAIR of units (j even, j+1): the low
// and high 32-bit halves decide units j and j+1; a unit is dropped iff its
// half < ceil(p * 2^32).  Keyed by (EST stream, step, token, unit pair).
__device__ __forceinline__ uint32_t drop_threshold32(float p) { return (uint32_t)ceil((double)p * 0x1p32); }
__device__ __forceinline__ void drop_scale2(uint64_t stream, int64_t step, int Te, int F, int tl, int j, float p,
                                            float keep, float* m0, float* m1) {  // j even
  if (p <= 0.f) {
    *m0 = *m1 = 1.f;
    return;
  }
  const uint64_t n = (((uint64_t)step * (uint64_t)Te + (uint64_t)tl) * (uint64_t)F + (uint64_t)j) >> 1;
  const uint64_t r = draw_raw(stream, n);
  const uint32_t t = drop_threshold32(p);
  *m0 = (uint32_t)r < t ? 0.f : keep;
  *m1 = (uint32_t)(r >> 32) < t ? 0.f : keep;
}

// GELU in its tanh form -- the activation of the original BERT code:
//   gelu(x) = 0.5 x (1 + tanh(c (x + 0.044715 x^3))),  c = sqrt(2/pi).
// tanh(u) = 1 - 2 / (1 + 2^(2u log2 e)) with the MUFU exp2 / fast reciprocal: absolute error ~1e-7,
// which is what 1 + tanh needs (no erf polynomial in the GEMM epilogue).
__device__ __forceinline__ float tanh_fast(float u) {
  return 1.f - __fdividef(2.f, 1.f + exp2f(2.8853900817779268f * u));
}
__device__ __forceinline__ float gelu(float x) {
  return 0.5f * x * (1.f + tanh_fast(0.7978845608028654f * (x + 0.044715f * x * x * x)));
}
__device__ __forceinline__ float gelu_grad(float x) {
  const float t = tanh_fast(0.7978845608028654f * (x + 0.044715f * x * x * x));
  return 0.5f * (1.f + t) + 0.5f * x * (1.f - t * t) * 0.7978845608028654f * (1.f + 0.134145f * x * x);
}
// Both from one tanh: the forward stores gelu'(h) for the backward (which then needs no transcendental).
// Written with explicit fused multiply-adds (the library builds with -fmad=false for the reference's
// fp64 path; here contraction is a deliberate, fixed choice) and the MUFU exp2 / reciprocal:
//   u = x (c + c k x^2),  t = 1 - 2 / (1 + 2^(2 log2(e) u)),  g = hx + hx t  (hx = x / 2),
//   g' = (1/2 + t/2) + hx (1 - t^2) (c + 3 c k x^2)
__device__ __forceinline__ float ex2_approx(float x) {
  float y;
  asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}
__device__ __forceinline__ void gelu_and_grad(float x, float* g, float* gd) {
  constexpr float C = 0.7978845608028654f, CK = C * 0.044715f, CK3 = 3.f * CK;
  const float x2 = __fmul_rn(x, x);
  const float u = __fmul_rn(x, __fmaf_rn(CK, x2, C));
  const float e = ex2_approx(__fmul_rn(2.8853900817779268f, u));
  const float t = __fsub_rn(1.f, __fdividef(2.f, __fadd_rn(1.f, e)));
  const float hx = __fmul_rn(0.5f, x);
  *g = __fmaf_rn(hx, t, hx);
  const float w = __fmul_rn(__fmul_rn(hx, __fmaf_rn(-t, t, 1.f)), __fmaf_rn(CK3, x2, C));
  *gd = __fmaf_rn(0.5f, t, __fadd_rn(0.5f, w));
}

}  // namespace ffn

// GEMM epilogue selector (bt_gemm.cu): what the epilogue warps do with a
// row-chunk of fp32 accumulators instead of storing them.
enum GemmEpiKind : int {
  EPI_STORE = 0,    // C = acc (fp32 or bf16)
  EPI_FFN_FWD = 1,  // h = acc + bias[j]: C = bf16(gelu'(h)) (kept for backward), out2 = bf16(dropout(gelu(h)))
  EPI_FFN_BWD = 2,  // C = bf16(acc * dropout_scale * aux[row][j])   (aux = the stored gelu'(h), bf16)
  EPI_BIAS = 3,     // C = acc + bias[j] (fp32 or bf16)
};
struct GemmEpi {
  int kind;
  const float* bias;          // [N] (FFN_FWD)
  const __nv_bfloat16* aux;   // [M][N] (FFN_BWD: gelu'(h))
  __nv_bfloat16* out2;        // [M][N] (FFN_FWD)
  uint64_t seed;
  int64_t step;
  int est_base, Te;           // row r belongs to EST est_base + r / Te
  float p;
};

}  // namespace bt
