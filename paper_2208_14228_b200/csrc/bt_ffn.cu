// bt_ffn.cu -- elementwise / layout kernels of the per-EST transformer FFN
// step (the C4 model-stack slice): the dense products run
// on the deterministic tcgen05 GEMM (bt_gemm.cu), the cross-EST gradient sum
// on the fixed-order reducer (bt_reduce.cu); this file holds what sits
// between them.  Every quantity is keyed by the EST's global rank and the
// step (counter-form splitmix64, as the reference keys dropout by rank,
// model.py:151-161), and every reduction has a fixed shape, so the bits do not
// depend on how ESTs are grouped into launches or mapped onto GPUs.
//
// Layout: the tokens of local EST e are rows [e*Te, (e+1)*Te) of X [T][D],
// H / A [T][F], Y [T][D]; bf16 activations, fp32 GEMM outputs.
#include <cuda_bf16.h>
#include <cuda_runtime.h>
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

// keep-scale of element (token tl, unit j) of EST eg at `step` (inverted dropout)
__device__ __forceinline__ float drop_scale(uint64_t stream, int64_t step, int Te, int F, int tl, int j, float p,
                                            float keep) {
  if (p <= 0.f) return 1.f;
  const uint64_t n = ((uint64_t)step * (uint64_t)Te + (uint64_t)tl) * (uint64_t)F + (uint64_t)j;
  return unit_float(draw_raw(stream, n)) < (double)p ? 0.f : keep;
}

__device__ __forceinline__ float gelu(float x) { return 0.5f * x * (1.f + erff(x * 0.70710678118654752f)); }
__device__ __forceinline__ float gelu_grad(float x) {
  return 0.5f * (1.f + erff(x * 0.70710678118654752f)) + x * 0.39894228040143268f * expf(-0.5f * x * x);
}

__global__ void data_kernel(uint64_t seed, int64_t step, int est_base, int E, int Te, int D, __nv_bfloat16* X,
                            float* target) {
  const int64_t n = (int64_t)E * Te * D;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    const int t = (int)(i / D), d = (int)(i - (int64_t)t * D);
    const int e = t / Te, tl = t - e * Te;
    const uint64_t idx = ((uint64_t)step * Te + tl) * (uint64_t)D + d;
    X[i] = __float2bfloat16_rn(uniform_pm1(derive3(TAG_FFN_X, seed, (uint64_t)(est_base + e)), idx));
    target[i] = 0.5f * uniform_pm1(derive3(TAG_FFN_Y, seed, (uint64_t)(est_base + e)), idx);
  }
}

// h = H32 + b1 -> Hpre (bf16, kept for backward); D = dropout(gelu(h)) (bf16)
__global__ void fwd_act_kernel(const float* __restrict__ H, const float* __restrict__ b1, uint64_t seed, int64_t step,
                               int est_base, int E, int Te, int F, float p, __nv_bfloat16* __restrict__ Hpre,
                               __nv_bfloat16* __restrict__ Dout) {
  const float keep = p < 1.f ? 1.f / (1.f - p) : 0.f;
  const int64_t n = (int64_t)E * Te * F;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    const int t = (int)(i / F), j = (int)(i - (int64_t)t * F);
    const int e = t / Te, tl = t - e * Te;
    const float h = H[i] + b1[j];
    Hpre[i] = __float2bfloat16_rn(h);
    const float m = drop_scale(derive3(TAG_FFN_DROP, seed, (uint64_t)(est_base + e)), step, Te, F, tl, j, p, keep);
    Dout[i] = __float2bfloat16_rn(gelu(h) * m);
  }
}

// diff = Y32 + b2 - target; dY = diff / Te (bf16); per-block loss partial
// sum 0.5*diff^2 over a fixed element range of one EST (fixed tree) -> part
constexpr int OUT_THREADS = 256, OUT_BLOCKS_PER_EST = 64;
__global__ void __launch_bounds__(OUT_THREADS) out_kernel(const float* __restrict__ Y, const float* __restrict__ b2,
                                                          const float* __restrict__ target, int Te, int D,
                                                          __nv_bfloat16* __restrict__ dY, float* __restrict__ part) {
  const int e = blockIdx.y, blk = blockIdx.x;
  const int64_t per_est = (int64_t)Te * D;
  const int64_t chunk = (per_est + OUT_BLOCKS_PER_EST - 1) / OUT_BLOCKS_PER_EST;
  const int64_t lo = blk * chunk, hi = min(per_est, lo + chunk);
  const float inv = 1.f / (float)Te;
  float acc = 0.f;
  for (int64_t k = lo + threadIdx.x; k < hi; k += OUT_THREADS) {  // thread-strided, ascending
    const int64_t i = (int64_t)e * per_est + k;
    const int d = (int)(k % D);
    const float diff = Y[i] + b2[d] - target[i];
    dY[i] = __float2bfloat16_rn(diff * inv);
    acc += 0.5f * diff * diff;
  }
  __shared__ float s[OUT_THREADS];
  s[threadIdx.x] = acc;
  __syncthreads();
  for (int w = OUT_THREADS / 2; w > 0; w >>= 1) {  // fixed pairwise tree
    if (threadIdx.x < w) s[threadIdx.x] += s[threadIdx.x + w];
    __syncthreads();
  }
  if (threadIdx.x == 0) part[e * OUT_BLOCKS_PER_EST + blk] = s[0];
}
__global__ void loss_final_kernel(const float* __restrict__ part, int E, int Te, float* __restrict__ loss) {
  const int e = blockIdx.x * blockDim.x + threadIdx.x;
  if (e >= E) return;
  float acc = 0.f;
  for (int b = 0; b < OUT_BLOCKS_PER_EST; ++b) acc += part[e * OUT_BLOCKS_PER_EST + b];  // ascending
  loss[e] = acc / (float)Te;
}

// dH = dropout'(dD32) * gelu'(Hpre)   (bf16)
__global__ void bwd_act_kernel(const float* __restrict__ dD, const __nv_bfloat16* __restrict__ Hpre, uint64_t seed,
                               int64_t step, int est_base, int E, int Te, int F, float p,
                               __nv_bfloat16* __restrict__ dH) {
  const float keep = p < 1.f ? 1.f / (1.f - p) : 0.f;
  const int64_t n = (int64_t)E * Te * F;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    const int t = (int)(i / F), j = (int)(i - (int64_t)t * F);
    const int e = t / Te, tl = t - e * Te;
    const float m = drop_scale(derive3(TAG_FFN_DROP, seed, (uint64_t)(est_base + e)), step, Te, F, tl, j, p, keep);
    dH[i] = __float2bfloat16_rn(dD[i] * m * gelu_grad(__bfloat162float(Hpre[i])));
  }
}

// out[e][c] = sum over r ascending of in[e][r][c]  (per-EST bias gradients)
__global__ void colsum_kernel(const __nv_bfloat16* __restrict__ in, int E, int R, int C, float* __restrict__ out) {
  const int64_t n = (int64_t)E * C;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    const int e = (int)(i / C), c = (int)(i - (int64_t)e * C);
    const __nv_bfloat16* p = in + (size_t)e * R * C + c;
    float acc = 0.f;
    for (int r = 0; r < R; ++r) acc += __bfloat162float(p[(size_t)r * C]);
    out[i] = acc;
  }
}

// out[e][c][r] = in[e][r][c]: 32x32 tiles through shared memory
template <class Tin>
__global__ void transpose_kernel(const Tin* __restrict__ in, int R, int C, __nv_bfloat16* __restrict__ out) {
  __shared__ float tile[32][33];
  const int e = blockIdx.z;
  const int r0 = blockIdx.y * 32, c0 = blockIdx.x * 32;
  const Tin* src = in + (size_t)e * R * C;
  __nv_bfloat16* dst = out + (size_t)e * R * C;
  for (int k = threadIdx.y; k < 32; k += blockDim.y) {
    const int r = r0 + k, c = c0 + threadIdx.x;
    if (r < R && c < C) tile[k][threadIdx.x] = (float)src[(size_t)r * C + c];
  }
  __syncthreads();
  for (int k = threadIdx.y; k < 32; k += blockDim.y) {
    const int c = c0 + k, r = r0 + threadIdx.x;
    if (r < R && c < C) dst[(size_t)c * R + r] = __float2bfloat16_rn(tile[threadIdx.x][k]);
  }
}

__global__ void cast_kernel(const float* __restrict__ in, int64_t n, __nv_bfloat16* __restrict__ out) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    out[i] = __float2bfloat16_rn(in[i]);
}

}  // namespace ffn

static int grid_for(int64_t n) {
  const int64_t g = (n + 255) / 256;
  return (int)(g > 148 * 16 ? 148 * 16 : (g < 1 ? 1 : g));
}
static int ok_or_cuda() { return cudaGetLastError() == cudaSuccess ? OK : ERR_CUDA; }

int ffn_data_launch(uint64_t seed, int64_t step, int est_base, int E, int Te, int D, void* X, float* target,
                    cudaStream_t s) {
  ffn::data_kernel<<<grid_for((int64_t)E * Te * D), 256, 0, s>>>(seed, step, est_base, E, Te, D,
                                                                   (__nv_bfloat16*)X, target);
  return ok_or_cuda();
}
int ffn_fwd_act_launch(const float* H, const float* b1, uint64_t seed, int64_t step, int est_base, int E, int Te,
                       int F, float p, void* Hpre, void* Dout, cudaStream_t s) {
  ffn::fwd_act_kernel<<<grid_for((int64_t)E * Te * F), 256, 0, s>>>(H, b1, seed, step, est_base, E, Te, F, p,
                                                                      (__nv_bfloat16*)Hpre, (__nv_bfloat16*)Dout);
  return ok_or_cuda();
}
int ffn_out_launch(const float* Y, const float* b2, const float* target, int E, int Te, int D, void* dY, float* part,
                   float* loss, cudaStream_t s) {
  ffn::out_kernel<<<dim3(ffn::OUT_BLOCKS_PER_EST, E), ffn::OUT_THREADS, 0, s>>>(Y, b2, target, Te, D,
                                                                                (__nv_bfloat16*)dY, part);
  ffn::loss_final_kernel<<<(E + 127) / 128, 128, 0, s>>>(part, E, Te, loss);
  return ok_or_cuda();
}
int ffn_bwd_act_launch(const float* dD, const void* Hpre, uint64_t seed, int64_t step, int est_base, int E, int Te,
                       int F, float p, void* dH, cudaStream_t s) {
  ffn::bwd_act_kernel<<<grid_for((int64_t)E * Te * F), 256, 0, s>>>(dD, (const __nv_bfloat16*)Hpre, seed, step,
                                                                      est_base, E, Te, F, p, (__nv_bfloat16*)dH);
  return ok_or_cuda();
}
int colsum_bf16_launch(const void* in, int E, int R, int C, float* out, cudaStream_t s) {
  ffn::colsum_kernel<<<grid_for((int64_t)E * C), 256, 0, s>>>((const __nv_bfloat16*)in, E, R, C, out);
  return ok_or_cuda();
}
int transpose_launch(const void* in, int in_f32, int E, int R, int C, void* out, cudaStream_t s) {
  const dim3 grid((C + 31) / 32, (R + 31) / 32, E), block(32, 8);
  if (in_f32)
    ffn::transpose_kernel<float><<<grid, block, 0, s>>>((const float*)in, R, C, (__nv_bfloat16*)out);
  else
    ffn::transpose_kernel<__nv_bfloat16><<<grid, block, 0, s>>>((const __nv_bfloat16*)in, R, C, (__nv_bfloat16*)out);
  return ok_or_cuda();
}
int cast_f32_bf16_launch(const float* in, int64_t n, void* out, cudaStream_t s) {
  ffn::cast_kernel<<<grid_for(n), 256, 0, s>>>(in, n, (__nv_bfloat16*)out);
  return ok_or_cuda();
}

}  // namespace bt
