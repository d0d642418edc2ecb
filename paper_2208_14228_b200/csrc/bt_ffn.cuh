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
// Every contraction is written out as an explicit fused multiply-add (the library builds with
// -fmad=false for the reference's fp64 path, and ptxas contracts the packed f32x2 forms below even when
// they are marked .rn -- so no separately rounded product may feed an addition here):
//   u = x (c + c k x^2),  r = rcp(1 + 2^(2 log2(e) u)),  t = fma(-r, 2, 1)  (= 1 - 2r exactly, = tanh u),
//   g = fma(hx, t, hx)  (hx = x / 2),  g' = fma(1/2, t, fma(hx (1 - t^2), c + 3 c k x^2, 1/2))
// with the MUFU exp2 / reciprocal: absolute error ~1e-7, which is what 1 + tanh needs.
__device__ __forceinline__ float ex2_approx(float x) {
  float y;
  asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}
__device__ __forceinline__ float rcp_approx(float x) {
  float y;
  asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}
__device__ __forceinline__ void gelu_and_grad(float x, float* g, float* gd) {
  constexpr float C = 0.7978845608028654f, CK = C * 0.044715f, CK3 = 3.f * CK;
  const float x2 = __fmul_rn(x, x);
  const float u = __fmul_rn(x, __fmaf_rn(CK, x2, C));
  const float e = ex2_approx(__fmul_rn(2.8853900817779268f, u));
  const float r = rcp_approx(__fadd_rn(1.f, e));
  const float t = __fmaf_rn(-r, 2.f, 1.f);
  const float hx = __fmul_rn(0.5f, x);
  *g = __fmaf_rn(hx, t, hx);
  const float w1 = __fmul_rn(hx, __fmaf_rn(-t, t, 1.f));
  *gd = __fmaf_rn(0.5f, t, __fmaf_rn(w1, __fmaf_rn(CK3, x2, C), 0.5f));
}

// Packed fp32 pairs (sm_100a FADD2 / FMUL2 / FFMA2: two IEEE round-to-nearest operations per
// instruction, the same bits as the scalar forms -- tools/check_f32x2.cu).  The GELU epilogue is
// FMA-pipe-bound, so the pair forms halve its issue count.
typedef unsigned long long f32x2;
__device__ __forceinline__ f32x2 pk2(float a, float b) {
  f32x2 r;
  asm("mov.b64 %0, {%1, %2};" : "=l"(r) : "f"(a), "f"(b));
  return r;
}
__device__ __forceinline__ float2 upk2(f32x2 r) {
  float2 f;
  asm("mov.b64 {%0, %1}, %2;" : "=f"(f.x), "=f"(f.y) : "l"(r));
  return f;
}
__device__ __forceinline__ f32x2 add2(f32x2 a, f32x2 b) {
  f32x2 r;
  asm("add.rn.f32x2 %0, %1, %2;" : "=l"(r) : "l"(a), "l"(b));
  return r;
}
__device__ __forceinline__ f32x2 sub2(f32x2 a, f32x2 b) {
  f32x2 r;
  asm("sub.rn.f32x2 %0, %1, %2;" : "=l"(r) : "l"(a), "l"(b));
  return r;
}
__device__ __forceinline__ f32x2 mul2(f32x2 a, f32x2 b) {
  f32x2 r;
  asm("mul.rn.f32x2 %0, %1, %2;" : "=l"(r) : "l"(a), "l"(b));
  return r;
}
__device__ __forceinline__ f32x2 fma2(f32x2 a, f32x2 b, f32x2 c) {
  f32x2 r;
  asm("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(r) : "l"(a), "l"(b), "l"(c));
  return r;
}
__device__ __forceinline__ uint32_t bf16x2_bits(f32x2 v) {
  const float2 f = upk2(v);
  const __nv_bfloat162 b = __floats2bfloat162_rn(f.x, f.y);
  return *(const uint32_t*)&b;
}
// gelu_and_grad on a pair, operation for operation (hence bit for bit -- tools/check_gelu2.cu)
__device__ __forceinline__ void gelu_and_grad2(f32x2 x, f32x2* g, f32x2* gd) {
  constexpr float C = 0.7978845608028654f, CK = C * 0.044715f, CK3 = 3.f * CK;
  const f32x2 kC = pk2(C, C), kCK = pk2(CK, CK), kCK3 = pk2(CK3, CK3), kL = pk2(2.8853900817779268f, 2.8853900817779268f);
  const f32x2 one = pk2(1.f, 1.f), mtwo = pk2(-2.f, -2.f), half = pk2(0.5f, 0.5f), mone = pk2(-1.f, -1.f);
  const f32x2 x2 = mul2(x, x);
  const f32x2 u = mul2(x, fma2(kCK, x2, kC));
  const float2 z = upk2(mul2(kL, u));
  const float2 d = upk2(add2(one, pk2(ex2_approx(z.x), ex2_approx(z.y))));
  const f32x2 r = pk2(rcp_approx(d.x), rcp_approx(d.y));
  const f32x2 t = fma2(r, mtwo, one);  // fma(-r, 2, 1): (-r) * 2 == r * (-2) exactly
  const f32x2 hx = mul2(half, x);
  *g = fma2(hx, t, hx);
  const f32x2 nt = mul2(t, mone);      // -t exactly
  const f32x2 w1 = mul2(hx, fma2(nt, t, one));
  *gd = fma2(half, t, fma2(w1, fma2(kCK3, x2, kC), half));
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
  float* colpart;             // FFN_BWD, optional: [M/32][N] column sums of the bf16 output over each 32-row
                              // block (fixed association), folded per gradient leaf by bt_colsum_fold
};

}  // namespace bt
