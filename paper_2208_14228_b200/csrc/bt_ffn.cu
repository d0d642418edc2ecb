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
#include "bt_ffn.cuh"

namespace bt {
namespace ffn {

// Row-oriented kernels: a block walks whole token rows (grid-stride), so the
// EST's counter stream is derived once per row, and each thread moves 8
// consecutive features with 16-byte loads/stores (dims are multiples of 128).
constexpr int ROW_THREADS = 128;

__device__ __forceinline__ void load8(const float* p, float* v) {
  const float4 a = *(const float4*)p, b = *(const float4*)(p + 4);
  v[0] = a.x; v[1] = a.y; v[2] = a.z; v[3] = a.w; v[4] = b.x; v[5] = b.y; v[6] = b.z; v[7] = b.w;
}
__device__ __forceinline__ void load8(const __nv_bfloat16* p, float* v) {
  const uint4 u = *(const uint4*)p;
  const __nv_bfloat162* h = (const __nv_bfloat162*)&u;
#pragma unroll
  for (int k = 0; k < 4; ++k) {
    const float2 f = __bfloat1622float2(h[k]);
    v[2 * k] = f.x;
    v[2 * k + 1] = f.y;
  }
}
__device__ __forceinline__ void store8(__nv_bfloat16* p, const float* v) {
  uint4 u;
  __nv_bfloat162* h = (__nv_bfloat162*)&u;
#pragma unroll
  for (int k = 0; k < 4; ++k) h[k] = __floats2bfloat162_rn(v[2 * k], v[2 * k + 1]);
  *(uint4*)p = u;
}

__global__ void __launch_bounds__(ROW_THREADS) data_kernel(uint64_t seed, int64_t step, int est_base, int Te, int D,
                                                           int rows, __nv_bfloat16* X, float* target) {
  for (int t = blockIdx.x; t < rows; t += gridDim.x) {
    const int e = t / Te, tl = t - e * Te;
    const uint64_t sx = derive3(TAG_FFN_X, seed, (uint64_t)(est_base + e));
    const uint64_t sy = derive3(TAG_FFN_Y, seed, (uint64_t)(est_base + e));
    const uint64_t row0 = ((uint64_t)step * Te + tl) * (uint64_t)D;
    for (int d0 = threadIdx.x * 8; d0 < D; d0 += ROW_THREADS * 8) {
      float xv[8], yv[8];
#pragma unroll
      for (int k = 0; k < 8; ++k) {
        xv[k] = uniform_pm1(sx, row0 + d0 + k);
        yv[k] = 0.5f * uniform_pm1(sy, row0 + d0 + k);
      }
      store8(X + (size_t)t * D + d0, xv);
      float4* tp = (float4*)(target + (size_t)t * D + d0);
      tp[0] = make_float4(yv[0], yv[1], yv[2], yv[3]);
      tp[1] = make_float4(yv[4], yv[5], yv[6], yv[7]);
    }
  }
}

// h = H32 + b1 -> Hpre = gelu'(h) (bf16, kept for backward); D = dropout(gelu(h)) (bf16)
__global__ void __launch_bounds__(ROW_THREADS) fwd_act_kernel(const float* __restrict__ H, const float* __restrict__ b1,
                                                              uint64_t seed, int64_t step, int est_base, int Te,
                                                              int F, int rows, float p, __nv_bfloat16* __restrict__ Hpre,
                                                              __nv_bfloat16* __restrict__ Dout) {
  const float keep = p < 1.f ? 1.f / (1.f - p) : 0.f;
  for (int t = blockIdx.x; t < rows; t += gridDim.x) {
    const int e = t / Te, tl = t - e * Te;
    const uint64_t sd = derive3(TAG_FFN_DROP, seed, (uint64_t)(est_base + e));
    for (int j0 = threadIdx.x * 8; j0 < F; j0 += ROW_THREADS * 8) {
      float h[8], b[8], d[8];
      load8(H + (size_t)t * F + j0, h);
      load8(b1 + j0, b);
#pragma unroll
      for (int k = 0; k < 8; k += 2) {
        float m0, m1;
        drop_scale2(sd, step, Te, F, tl, j0 + k, p, keep, &m0, &m1);
        float g0, g1;
        gelu_and_grad(h[k] + b[k], &g0, &h[k]);
        gelu_and_grad(h[k + 1] + b[k + 1], &g1, &h[k + 1]);
        d[k] = g0 * m0;
        d[k + 1] = g1 * m1;
      }
      store8(Hpre + (size_t)t * F + j0, h);
      store8(Dout + (size_t)t * F + j0, d);
    }
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

// dH = dropout'(dD32) * Hpre   (Hpre = the stored gelu'(h); bf16)
__global__ void __launch_bounds__(ROW_THREADS) bwd_act_kernel(const float* __restrict__ dD,
                                                              const __nv_bfloat16* __restrict__ Hpre, uint64_t seed,
                                                              int64_t step, int est_base, int Te, int F, int rows,
                                                              float p, __nv_bfloat16* __restrict__ dH) {
  const float keep = p < 1.f ? 1.f / (1.f - p) : 0.f;
  for (int t = blockIdx.x; t < rows; t += gridDim.x) {
    const int e = t / Te, tl = t - e * Te;
    const uint64_t sd = derive3(TAG_FFN_DROP, seed, (uint64_t)(est_base + e));
    for (int j0 = threadIdx.x * 8; j0 < F; j0 += ROW_THREADS * 8) {
      float g[8], h[8];
      load8(dD + (size_t)t * F + j0, g);
      load8(Hpre + (size_t)t * F + j0, h);
#pragma unroll
      for (int k = 0; k < 8; k += 2) {
        float m0, m1;
        drop_scale2(sd, step, Te, F, tl, j0 + k, p, keep, &m0, &m1);
        g[k] = g[k] * m0 * h[k];
        g[k + 1] = g[k + 1] * m1 * h[k + 1];
      }
      store8(dH + (size_t)t * F + j0, g);
    }
  }
}

// out[e][c] = sum over r of in[e][r][c] (per-EST / per-leaf bias gradients), in a fixed association:
// ascending 64-row chunks (COLSUM_ROWS, fixed: part of the reduction's shape) are summed ascending into
// partials (pass 1, parallel over chunks x columns), then the partials are summed in chunk order
// (pass 2).  Same bits for any grid.
constexpr int COLSUM_ROWS = 64;
__global__ void colsum_part_kernel(const __nv_bfloat16* __restrict__ in, int E, int R, int C,
                                   float* __restrict__ part) {
  const int cpt = C / 8, chunks = (R + COLSUM_ROWS - 1) / COLSUM_ROWS;
  const int64_t n = (int64_t)E * chunks * cpt;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    const int c0 = (int)(i % cpt) * 8;
    const int64_t ek = i / cpt;
    const int k = (int)(ek % chunks), e = (int)(ek / chunks);
    const int r0 = k * COLSUM_ROWS, r1 = min(R, r0 + COLSUM_ROWS);
    const __nv_bfloat16* p = in + (size_t)e * R * C + c0;
    float acc[8] = {0, 0, 0, 0, 0, 0, 0, 0};
#pragma unroll 4
    for (int r = r0; r < r1; ++r) {
      float v[8];
      load8(p + (size_t)r * C, v);
#pragma unroll
      for (int q = 0; q < 8; ++q) acc[q] += v[q];
    }
    float4* o = (float4*)(part + ((size_t)e * chunks + k) * C + c0);
    o[0] = make_float4(acc[0], acc[1], acc[2], acc[3]);
    o[1] = make_float4(acc[4], acc[5], acc[6], acc[7]);
  }
}
// Fold of the chunk partials per (EST / leaf, column): the chunks in 8 contiguous groups of q = ceil(chunks/8),
// each group summed in chunk order by its own warp (32 columns per block), then the groups in order -- a fixed
// association for every grid (for chunks <= 8 exactly the sequential sum).  A sequential sum per column
// left the fold latency-bound on a chain of loads (~10 us per launch at 128 chunks).
__global__ void __launch_bounds__(256) colsum_final_kernel(const float* __restrict__ part, int E, int chunks, int C,
                                                           float* __restrict__ out, int64_t ostride) {
  __shared__ float sp[8][33];
  const int cl = threadIdx.x & 31, g = threadIdx.x >> 5;
  const int64_t ncb = (C + 31) / 32;
  const int q = (chunks + 7) / 8, ng = (chunks + q - 1) / q;
  for (int64_t b = blockIdx.x; b < (int64_t)E * ncb; b += gridDim.x) {
    const int e = (int)(b / ncb), c = (int)(b - (int64_t)e * ncb) * 32 + cl;
    const int k0 = g * q, k1 = min(chunks, k0 + q);
    float acc = 0.f;
    if (c < C && k0 < k1) {
      const float* pc = part + ((size_t)e * chunks) * C + c;
      acc = pc[(size_t)k0 * C];
      int k = k0 + 1;
      for (; k + 4 <= k1; k += 4) {
        float v[4];
#pragma unroll
        for (int j = 0; j < 4; ++j) v[j] = pc[(size_t)(k + j) * C];
#pragma unroll
        for (int j = 0; j < 4; ++j) acc += v[j];
      }
      for (; k < k1; ++k) acc += pc[(size_t)k * C];
    }
    sp[g][cl] = acc;
    __syncthreads();
    if (g == 0 && c < C) {
      float t = sp[0][cl];
      for (int gg = 1; gg < ng; ++gg) t += sp[gg][cl];
      out[(size_t)e * ostride + c] = t;
    }
    __syncthreads();
  }
}

// out[e][c][r] = in[e][r][c]: 64x64 tiles through shared memory, 4-byte
// (two-element) accesses on both sides
template <class Tin>
__global__ void __launch_bounds__(256) transpose_kernel(const Tin* __restrict__ in, int R, int C,
                                                        __nv_bfloat16* __restrict__ out) {
  __shared__ float tile[64][65];
  const int e = blockIdx.z;
  const int r0 = blockIdx.y * 64, c0 = blockIdx.x * 64;
  const Tin* src = in + (size_t)e * R * C;
  __nv_bfloat16* dst = out + (size_t)e * R * C;
  const int tx = threadIdx.x & 31, ty = threadIdx.x >> 5;  // 32 x 8
  for (int k = ty; k < 64; k += 8) {
    const int r = r0 + k, c = c0 + 2 * tx;
    if (r < R && c + 1 < C) {
      float2 v;
      if constexpr (sizeof(Tin) == 4) v = *(const float2*)(src + (size_t)r * C + c);
      else v = __bfloat1622float2(*(const __nv_bfloat162*)(src + (size_t)r * C + c));
      tile[k][2 * tx] = v.x;
      tile[k][2 * tx + 1] = v.y;
    }
  }
  __syncthreads();
  for (int k = ty; k < 64; k += 8) {
    const int c = c0 + k, r = r0 + 2 * tx;
    if (c < C && r + 1 < R)
      *(__nv_bfloat162*)(dst + (size_t)c * R + r) = __floats2bfloat162_rn(tile[2 * tx][k], tile[2 * tx + 1][k]);
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

int colsum_bf16_strided_launch(const void* in, int E, int R, int C, float* out, int64_t ostride, float* scratch,
                               cudaStream_t s);
static int row_grid(int rows) { return rows < 148 * 16 ? rows : 148 * 16; }

int ffn_data_launch(uint64_t seed, int64_t step, int est_base, int E, int Te, int D, void* X, float* target,
                    cudaStream_t s) {
  if (D % 8) return ERR_INPUT;
  ffn::data_kernel<<<row_grid(E * Te), ffn::ROW_THREADS, 0, s>>>(seed, step, est_base, Te, D, E * Te,
                                                                    (__nv_bfloat16*)X, target);
  return ok_or_cuda();
}
int ffn_fwd_act_launch(const float* H, const float* b1, uint64_t seed, int64_t step, int est_base, int E, int Te,
                       int F, float p, void* Hpre, void* Dout, cudaStream_t s) {
  if (F % 8) return ERR_INPUT;
  ffn::fwd_act_kernel<<<row_grid(E * Te), ffn::ROW_THREADS, 0, s>>>(H, b1, seed, step, est_base, Te, F, E * Te, p,
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
  if (F % 8) return ERR_INPUT;
  ffn::bwd_act_kernel<<<row_grid(E * Te), ffn::ROW_THREADS, 0, s>>>(dD, (const __nv_bfloat16*)Hpre, seed, step,
                                                                       est_base, Te, F, E * Te, p, (__nv_bfloat16*)dH);
  return ok_or_cuda();
}
int colsum_bf16_launch(const void* in, int E, int R, int C, float* out, float* scratch, cudaStream_t s) {
  return colsum_bf16_strided_launch(in, E, R, C, out, C, scratch, s);
}
int colsum_bf16_strided_launch(const void* in, int E, int R, int C, float* out, int64_t ostride, float* scratch,
                               cudaStream_t s) {
  if (C % 8) return ERR_INPUT;
  const int chunks = (R + ffn::COLSUM_ROWS - 1) / ffn::COLSUM_ROWS;
  float* part = scratch;  // E * ceil(R / 64) * C partials
  bool own = false;
  if (!part) {
    if (cudaMallocAsync((void**)&part, sizeof(float) * (size_t)E * chunks * C, s) != cudaSuccess) return ERR_CUDA;
    own = true;
  }
  ffn::colsum_part_kernel<<<grid_for((int64_t)E * chunks * C / 8), 256, 0, s>>>((const __nv_bfloat16*)in, E, R, C,
                                                                               part);
  ffn::colsum_final_kernel<<<grid_for((int64_t)E * ((C + 31) / 32) * 256), 256, 0, s>>>(part, E, chunks, C, out,
                                                                                      ostride);
  if (own) cudaFreeAsync(part, s);
  return ok_or_cuda();
}
int colsum_fold_launch(const float* part, int E, int chunks, int C, float* out, int64_t ostride, cudaStream_t s) {
  ffn::colsum_final_kernel<<<grid_for((int64_t)E * ((C + 31) / 32) * 256), 256, 0, s>>>(part, E, chunks, C, out,
                                                                                      ostride);
  return ok_or_cuda();
}
int transpose_launch(const void* in, int in_f32, int E, int R, int C, void* out, cudaStream_t s) {
  if (R % 2 || C % 2) return ERR_INPUT;
  const dim3 grid((C + 63) / 64, (R + 63) / 64, E);
  if (in_f32)
    ffn::transpose_kernel<float><<<grid, 256, 0, s>>>((const float*)in, R, C, (__nv_bfloat16*)out);
  else
    ffn::transpose_kernel<__nv_bfloat16><<<grid, 256, 0, s>>>((const __nv_bfloat16*)in, R, C, (__nv_bfloat16*)out);
  return ok_or_cuda();
}
int cast_f32_bf16_launch(const float* in, int64_t n, void* out, cudaStream_t s) {
  ffn::cast_kernel<<<grid_for(n), 256, 0, s>>>(in, n, (__nv_bfloat16*)out);
  return ok_or_cuda();
}

}  // namespace bt
