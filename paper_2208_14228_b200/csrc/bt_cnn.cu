// bt_cnn.cu -- the kernels between the GEMMs of a per-EST ResNet-18 step with
// BatchNorm (C3, BASELINE.json configs[2]).  No reference
// implementation exists for this model.  The EasyScale contract:
// every EST normalises with the statistics of its OWN micro-batch and keeps its
// OWN BatchNorm running statistics (an HBM slot indexed by EST rank, moved
// with the EST on an elastic rescale), its data are keyed by (seed, EST rank,
// EST sampler cursor), and every reduction has a shape fixed by the EST's data
// -- so the bits never depend on which ESTs share a launch or a GPU.
//
// Layout: NHWC bf16 activations; the images of local EST e are n in
// [e*B, (e+1)*B), so its rows (n, h, w) are one contiguous block of B*H*W rows.
// Convolutions are GEMMs on the deterministic tcgen05 kernels (bt_gemm.cu; implicit im2col
// operands by TMA, or the explicit im2col below -- the same tiles and K order):
//   forward  z = im2col(x) . W^T        (K = KH*KW*Ci, ordered (kh, kw, ci))
//   dX       stride 1: a forward convolution of dz with the tap-reversed filter;
//            stride 2: four output parity classes, each a stride-1 convolution of
//            dz with its class filter (filter_taps_kernel), interleaved by
//            add_s2_kernel (no scatter, no atomics, no zero products)
//   dW_e     = dz_e^T im2col(x)_e       (MN-major batched GEMM, one per EST split)
#include <cuda_bf16.h>
#include <cuda_runtime.h>
#include <stdint.h>

#include "bt_common.cuh"

namespace bt {
namespace cnn {

constexpr uint64_t TAG_CNN_X = 0x434e'4e5f'5844'4154ull;      // "CNN_XDAT"
constexpr uint64_t TAG_CNN_LABEL = 0x434e'4e5f'4c41'424cull;  // "CNN_LABL"
// rows per column-statistics partial: a function of the channel count and the mode only (part of the
// reduction's shape, the same for every EST mapping); sized for the HBM pass at ResNet-18 shapes
inline int chunk_rows(int C, int mode) { return mode == 0 && C <= 64 ? 1024 : 256; }

__device__ __forceinline__ void ld8(const __nv_bfloat16* p, float* v) {
  const uint4 u = *(const uint4*)p;
  const __nv_bfloat162* h = (const __nv_bfloat162*)&u;
#pragma unroll
  for (int k = 0; k < 4; ++k) {
    const float2 f = __bfloat1622float2(h[k]);
    v[2 * k] = f.x;
    v[2 * k + 1] = f.y;
  }
}
__device__ __forceinline__ void ldf8(const float* p, float* v) {  // 32-byte aligned
  const float4 a = __ldg((const float4*)p), b = __ldg((const float4*)p + 1);
  v[0] = a.x, v[1] = a.y, v[2] = a.z, v[3] = a.w, v[4] = b.x, v[5] = b.y, v[6] = b.z, v[7] = b.w;
}
__device__ __forceinline__ void st8(__nv_bfloat16* p, const float* v) {
  uint4 u;
  __nv_bfloat162* h = (__nv_bfloat162*)&u;
#pragma unroll
  for (int k = 0; k < 4; ++k) h[k] = __floats2bfloat162_rn(v[2 * k], v[2 * k + 1]);
  *(uint4*)p = u;
}

// ---------------------------------------------------------------- data
// images [E*B][32][32][8] bf16 (channels 3..7 zero), labels [E*B]: image nl of EST e at its sampler
// cursor c = cursor[e]: pixel draws (TAG_CNN_X, seed, EST) at (c*B + nl)*3072 + (h*32 + w)*3 + ch,
// label (TAG_CNN_LABEL, seed, EST) draw c*B + nl mod 10
__global__ void data_kernel(uint64_t seed, const int64_t* __restrict__ cursor, int est_base, int B, int E,
                            __nv_bfloat16* __restrict__ x, int32_t* __restrict__ labels) {
  const int64_t n = (int64_t)E * B * 1024;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    const int img = (int)(i >> 10), pix = (int)(i & 1023);
    const int e = img / B, nl = img - e * B;
    const uint64_t c = (uint64_t)cursor[e];
    const uint64_t sx = derive3(TAG_CNN_X, seed, (uint64_t)(est_base + e));
    const uint64_t base = ((c * B + nl) * 1024 + pix) * 3;
    float v[8] = {0, 0, 0, 0, 0, 0, 0, 0};
#pragma unroll
    for (int ch = 0; ch < 3; ++ch) v[ch] = (float)(unit_float(draw_raw(sx, base + ch)) * 2.0 - 1.0);
    st8(x + i * 8, v);
    if (pix == 0) {
      const uint64_t sl = derive3(TAG_CNN_LABEL, seed, (uint64_t)(est_base + e));
      labels[img] = (int32_t)(draw_raw(sl, c * B + nl) % 10u);
    }
  }
}

// ---------------------------------------------------------------- im2col
// col[(n, ho, wo)][(kh, kw, c)] (8 channels per thread, 16-byte moves).
// forward:     source (ho*s - p + kh, wo*s - p + kw) of x [N][Hs][Ws][C]
// transposed:  (the dX gather of a stride-s convolution) output grid = the forward input grid;
//              source ((ho + p - kh)/s, (wo + p - kw)/s) of dz [N][Hs][Ws][C] when exact and in range
struct ColArgs {
  const __nv_bfloat16* src;
  __nv_bfloat16* col;
  int N, Hs, Ws, C, Ho, Wo, KH, KW, s, p, transposed;
};
// One warp per output row (its (image, ho, wo) decoded once); lanes walk the row's K8 16-byte
// chunks -- coalesced stores, contiguous 16-byte reads per tap -- with shift/mask decoding (C/8 a
// power of two, KW <= 3): the kernel is store-bandwidth-bound rather than integer-bound.
// ROWPACK (K8 < 32, e.g. the 8-channel stem): thread per (row, chunk) item instead, so short rows do
// not leave most of a warp idle; the stores stay contiguous across rows.
template <bool ROWPACK>
__global__ void __launch_bounds__(256) im2col_kernel(const ColArgs a, int lcg) {
  const int cg = 1 << lcg, K8 = a.KH * a.KW * cg;
  const int rows = a.N * a.Ho * a.Wo, HoWo = a.Ho * a.Wo;
  const int lane = threadIdx.x & 31;
  const int64_t items = ROWPACK ? (int64_t)rows * K8 : rows;
  const int64_t first = ROWPACK ? blockIdx.x * (int64_t)blockDim.x + threadIdx.x
                                : (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  const int64_t stride = ROWPACK ? (int64_t)gridDim.x * blockDim.x : ((int64_t)gridDim.x * blockDim.x) >> 5;
  for (int64_t it = first; it < items; it += stride) {
    const int r = ROWPACK ? (int)(it / K8) : (int)it;
    const int img = r / HoWo, pix = r - img * HoWo;
    const int ho = pix / a.Wo, wo = pix - ho * a.Wo;
    const __nv_bfloat16* src = a.src + (size_t)img * a.Hs * a.Ws * a.C;
    uint4* dst = (uint4*)(a.col + (size_t)r * K8 * 8);
    const int kb = ROWPACK ? (int)(it - (int64_t)r * K8) : lane;
    for (int k8 = kb; k8 < K8; k8 += ROWPACK ? K8 : 32) {
      const int t = k8 >> lcg, c8 = k8 & (cg - 1);
      const int kh = a.KW == 3 ? (t * 11) >> 5 : (a.KW == 2 ? t >> 1 : t), kw = t - kh * a.KW;  // t / 3 for t < 9
      int hi, wi;
      bool ok;
      if (!a.transposed) {
        hi = ho * a.s - a.p + kh;
        wi = wo * a.s - a.p + kw;
        ok = true;
      } else {
        const int hn = ho + a.p - kh, wn = wo + a.p - kw;
        ok = hn >= 0 && wn >= 0 && ((hn | wn) & (a.s - 1)) == 0;  // s in {1, 2}
        hi = hn >> (a.s - 1);
        wi = wn >> (a.s - 1);
      }
      ok = ok && hi >= 0 && hi < a.Hs && wi >= 0 && wi < a.Ws;
      uint4 v = make_uint4(0, 0, 0, 0);
      if (ok) v = *(const uint4*)(src + ((size_t)hi * a.Ws + wi) * a.C + c8 * 8);
      dst[k8] = v;
    }
  }
}

// ---------------------------------------------------------------- BatchNorm
// Column statistics per EST over fixed chunk_rows(C, mode)-row chunks: block = (chunk k, 64-channel slice, local EST
// e); thread = (row lane, 8-channel group); rows walked in order, lanes combined in lane order.
//   mode 0: sum (z - k), sum (z - k)^2   (one pass; k = the EST's first row, a per-channel shift
//           that keeps the variance free of cancellation)
//   mode 2: sum g, sum g * xhat         (g = dy * [y > 0], xhat = (z - mean) * rstd)
struct StatArgs {
  const __nv_bfloat16* z;     // conv output (pre-BN)
  const __nv_bfloat16* dy;    // mode 2: gradient of the block/ReLU output
  const __nv_bfloat16* y;     // mode 2: the ReLU output (mask)
  const float* mean;          // [E][C] (mode 2)
  const float* rstd;          // [E][C] (mode 2)
  float* part;                // [E][chunks][2][C]
  int C, R, mode, chunk;      // R = rows per EST, chunk = chunk_rows(C)
};
template <int MODE>
__global__ void __launch_bounds__(256, 4) stats_kernel(const StatArgs a) {
  __shared__ float st_smem[8 * 2 * 64];  // [warps][2][SW]
  const int k = blockIdx.x, e = blockIdx.z, chunks = gridDim.x;
  const int SW = min(a.C, 64), cg = SW / 8, lanes = 256 / cg;
  const int lane = threadIdx.x / cg, cl = (threadIdx.x % cg) * 8, c0 = blockIdx.y * 64 + cl;
  float s0[8] = {0, 0, 0, 0, 0, 0, 0, 0}, s1[8] = {0, 0, 0, 0, 0, 0, 0, 0};
  float m[8], r[8];
  if (MODE == 0) ld8(a.z + (size_t)e * a.R * a.C + c0, m);  // shift k = row 0 of the EST
  else
    for (int q = 0; q < 8; ++q) m[q] = a.mean[(size_t)e * a.C + c0 + q];
  if (MODE == 2)
    for (int q = 0; q < 8; ++q) r[q] = a.rstd[(size_t)e * a.C + c0 + q];
  const int r1 = min(a.R, (k + 1) * a.chunk);
#pragma unroll 4
  for (int row = k * a.chunk + lane; row < r1; row += lanes) {
    const size_t off = ((size_t)e * a.R + row) * a.C + c0;
    float zv[8];
    ld8(a.z + off, zv);
    if (MODE == 0) {
#pragma unroll
      for (int q = 0; q < 8; ++q) {
        const float d = zv[q] - m[q];
        s0[q] += d;
        s1[q] += d * d;
      }
    } else {
      float dv[8], yv[8];
      ld8(a.dy + off, dv);
      ld8(a.y + off, yv);
#pragma unroll
      for (int q = 0; q < 8; ++q) {
        const float g = yv[q] > 0.f ? dv[q] : 0.f;
        s0[q] += g;
        s1[q] += g * ((zv[q] - m[q]) * r[q]);
      }
    }
  }
  // lanes of a warp (32 / cg row lanes) combined by a fixed butterfly, then the 8 warps in order
  for (int o = cg; o < 32; o <<= 1)
#pragma unroll
    for (int q = 0; q < 8; ++q) {
      s0[q] += __shfl_xor_sync(0xffffffffu, s0[q], o);
      s1[q] += __shfl_xor_sync(0xffffffffu, s1[q], o);
    }
  const int warp = threadIdx.x >> 5;
  if ((threadIdx.x & 31) < cg)
#pragma unroll
    for (int q = 0; q < 8; ++q) {
      st_smem[(warp * 2 + 0) * SW + cl + q] = s0[q];
      st_smem[(warp * 2 + 1) * SW + cl + q] = s1[q];
    }
  __syncthreads();
  float* out = a.part + ((size_t)e * chunks + k) * 2 * a.C + blockIdx.y * 64;
  for (int i = threadIdx.x; i < 2 * SW; i += 256) {
    const int j = i / SW, c = i - j * SW;
    float acc = st_smem[j * SW + c];
#pragma unroll
    for (int w = 1; w < 8; ++w) acc += st_smem[(w * 2 + j) * SW + c];
    out[(size_t)j * a.C + c] = acc;
  }
}

// Fold the chunk partials in chunk order.  mode 0: d = S/R, mean = k + d, var = Q/R - d^2, rstd, and
// the EST's running statistics (slot): rm = 0.9 rm + 0.1 mean, rv = 0.9 rv + 0.1 var * R/(R-1).
// mode 2: (sum g, sum g*xhat) -> out0 / out1 (and dbeta / dgamma into the EST's gradient slot).
struct FoldArgs {
  const float* part;
  float* out0;      // mode 0: mean [E][C]; mode 2: sum g [E][C]
  float* out1;      // mode 0: rstd [E][C]; mode 2: sum g*xhat [E][C]
  const __nv_bfloat16* z;  // mode 0: the shift rows
  float* run_mean;  // slot [E] x stride
  float* run_var;
  int64_t run_stride;
  float* dgamma;    // grad slot of EST e at + e*grad_stride
  float* dbeta;
  int64_t grad_stride;
  int C, R, E, chunks, mode;
  float eps;
};
// One warp per (EST, channel): lane l sums chunks l, l+32, ... in order, then a fixed xor butterfly
// (every lane ends with the same bits: IEEE addition commutes).
__global__ void fold_kernel(const FoldArgs a) {
  const int64_t n = (int64_t)a.E * a.C;
  const int lane = threadIdx.x & 31;
  for (int64_t i = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5; i < n;
       i += ((int64_t)gridDim.x * blockDim.x) >> 5) {
    const int e = (int)(i / a.C), c = (int)(i - (int64_t)e * a.C);
    const float* p = a.part + (size_t)e * a.chunks * 2 * a.C + c;
    float s0 = 0.f, s1 = 0.f;
    for (int k = lane; k < a.chunks; k += 32) {
      s0 += p[(size_t)k * 2 * a.C];
      s1 += p[(size_t)k * 2 * a.C + a.C];
    }
#pragma unroll
    for (int o = 16; o; o >>= 1) {
      s0 += __shfl_xor_sync(0xffffffffu, s0, o);
      s1 += __shfl_xor_sync(0xffffffffu, s1, o);
    }
    if (lane) continue;
    if (a.mode == 0) {
      const float k = __bfloat162float(a.z[(size_t)e * a.R * a.C + c]);
      const float d = s0 / (float)a.R;
      const float mean = k + d, var = fmaxf(s1 / (float)a.R - d * d, 0.f);
      a.out0[i] = mean;
      a.out1[i] = 1.f / sqrtf(var + a.eps);
      float* rm = a.run_mean + (size_t)e * a.run_stride + c;
      float* rv = a.run_var + (size_t)e * a.run_stride + c;
      *rm = 0.9f * *rm + 0.1f * mean;
      *rv = 0.9f * *rv + 0.1f * (var * ((float)a.R / (float)(a.R - 1)));
    } else {
      a.out0[i] = s0;
      a.out1[i] = s1;
      a.dbeta[(size_t)e * a.grad_stride + c] = s0;
      a.dgamma[(size_t)e * a.grad_stride + c] = s1;
    }
  }
}

// Block = (local EST e, a span of `rows_per` of that EST's rows, sized on the host for ~4 blocks per SM);
// the EST's per-channel parameters are staged in shared memory once per block and each thread walks its
// 8-channel group down the span's rows, BN_UNROLL rows' loads in flight at a time.  The per-element
// arithmetic is unchanged.
constexpr int BN_THREADS = 256, BN_UNROLL = 4;
__device__ __forceinline__ void cvt8(const uint4& u, float* v) {
  const __nv_bfloat162* h = (const __nv_bfloat162*)&u;
#pragma unroll
  for (int k = 0; k < 4; ++k) {
    const float2 f = __bfloat1622float2(h[k]);
    v[2 * k] = f.x;
    v[2 * k + 1] = f.y;
  }
}
__device__ __forceinline__ void lds8(const float* p, float* v) {
  const float4 a = *(const float4*)p, b = *(const float4*)(p + 4);
  v[0] = a.x, v[1] = a.y, v[2] = a.z, v[3] = a.w, v[4] = b.x, v[5] = b.y, v[6] = b.z, v[7] = b.w;
}

// y = [relu](gamma * (z - mean) * rstd + beta [+ res])   (bf16, 8 channels per thread)
__global__ void __launch_bounds__(BN_THREADS, 2) bn_apply_kernel(const __nv_bfloat16* __restrict__ z,
                                                              const __nv_bfloat16* __restrict__ res,
                                                              const float* __restrict__ mean,
                                                              const float* __restrict__ rstd,
                                                              const float* __restrict__ gamma,
                                                              const float* __restrict__ beta, int C, int R, int relu,
                                                              int rows_per, __nv_bfloat16* __restrict__ y) {
  extern __shared__ __align__(16) float bnp[];  // [4][C]: mean, rstd, gamma, beta of this block's EST
  const int e = blockIdx.y;
  for (int i = threadIdx.x; i < C; i += BN_THREADS) {
    bnp[i] = mean[(size_t)e * C + i];
    bnp[C + i] = rstd[(size_t)e * C + i];
    bnp[2 * C + i] = gamma[i];
    bnp[3 * C + i] = beta[i];
  }
  __syncthreads();
  const int cg = C / 8, lanes = BN_THREADS / cg;  // C in {64 .. 512}: cg divides 256
  const int c0 = (threadIdx.x % cg) * 8, lane = threadIdx.x / cg;
  const int r0 = blockIdx.x * rows_per, r1 = min(R, r0 + rows_per);
  float mv[8], sv[8], gv[8], bv[8];
  lds8(bnp + c0, mv);
  lds8(bnp + C + c0, sv);
  lds8(bnp + 2 * C + c0, gv);
  lds8(bnp + 3 * C + c0, bv);
  const size_t base = (size_t)e * R * C + c0;
  for (int r = r0 + lane; r < r1; r += BN_UNROLL * lanes) {
    uint4 zr[BN_UNROLL], rr_[BN_UNROLL];  // raw bf16: the loads of all unrolled rows in flight at once
#pragma unroll
    for (int u = 0; u < BN_UNROLL; ++u) {
      const int rr = r + u * lanes;
      if (rr < r1) {
        zr[u] = *(const uint4*)(z + base + (size_t)rr * C);
        if (res) rr_[u] = *(const uint4*)(res + base + (size_t)rr * C);
      }
    }
#pragma unroll
    for (int u = 0; u < BN_UNROLL; ++u) {
      const int rr = r + u * lanes;
      if (rr >= r1) continue;
      float o[8], zv[1][8], rv[1][8];
      cvt8(zr[u], zv[0]);
      if (res) cvt8(rr_[u], rv[0]);
#pragma unroll
      for (int q = 0; q < 8; ++q) {
        float v = gv[q] * ((zv[0][q] - mv[q]) * sv[q]) + bv[q];
        if (res) v += rv[0][q];
        o[q] = (relu && !(v > 0.f)) ? 0.f : v;
      }
      st8(y + base + (size_t)rr * C, o);
    }
  }
}

// dz = gamma * rstd * (g - S_g / R - xhat * S_gx / R),  g = dy * [y > 0]
__global__ void __launch_bounds__(BN_THREADS, 2) bn_bwd_kernel(const __nv_bfloat16* __restrict__ z,
                                                            const __nv_bfloat16* __restrict__ dy,
                                                            const __nv_bfloat16* __restrict__ y,
                                                            const float* __restrict__ mean,
                                                            const float* __restrict__ rstd,
                                                            const float* __restrict__ sg,
                                                            const float* __restrict__ sgx,
                                                            const float* __restrict__ gamma, int C, int R,
                                                            int rows_per, __nv_bfloat16* __restrict__ dz) {
  extern __shared__ __align__(16) float bnp[];  // [5][C]: mean, rstd, S_g, S_gx, gamma
  const int e = blockIdx.y;
  for (int i = threadIdx.x; i < C; i += BN_THREADS) {
    const size_t ec = (size_t)e * C + i;
    bnp[i] = mean[ec];
    bnp[C + i] = rstd[ec];
    bnp[2 * C + i] = sg[ec];
    bnp[3 * C + i] = sgx[ec];
    bnp[4 * C + i] = gamma[i];
  }
  __syncthreads();
  const float invR = 1.f / (float)R;
  const int cg = C / 8, lanes = BN_THREADS / cg;
  const int c0 = (threadIdx.x % cg) * 8, lane = threadIdx.x / cg;
  const int r0 = blockIdx.x * rows_per, r1 = min(R, r0 + rows_per);
  float mv[8], sv[8], av[8], bv[8], gv[8];
  lds8(bnp + c0, mv);
  lds8(bnp + C + c0, sv);
  lds8(bnp + 2 * C + c0, av);
  lds8(bnp + 3 * C + c0, bv);
  lds8(bnp + 4 * C + c0, gv);
  const size_t base = (size_t)e * R * C + c0;
  for (int r = r0 + lane; r < r1; r += BN_UNROLL * lanes) {
    uint4 zr[BN_UNROLL], dr[BN_UNROLL], yr[BN_UNROLL];  // raw bf16: all unrolled rows' loads in flight
#pragma unroll
    for (int u = 0; u < BN_UNROLL; ++u) {
      const int rr = r + u * lanes;
      if (rr < r1) {
        const size_t off = base + (size_t)rr * C;
        zr[u] = *(const uint4*)(z + off);
        dr[u] = *(const uint4*)(dy + off);
        yr[u] = *(const uint4*)(y + off);
      }
    }
#pragma unroll
    for (int u = 0; u < BN_UNROLL; ++u) {
      const int rr = r + u * lanes;
      if (rr >= r1) continue;
      float o[8], zv[8], dv[8], yv[8];
      cvt8(zr[u], zv);
      cvt8(dr[u], dv);
      cvt8(yr[u], yv);
#pragma unroll
      for (int q = 0; q < 8; ++q) {
        const float g = yv[q] > 0.f ? dv[q] : 0.f;
        const float xh = (zv[q] - mv[q]) * sv[q];
        o[q] = gv[q] * sv[q] * (g - av[q] * invR - xh * (bv[q] * invR));
      }
      st8(dz + base + (size_t)rr * C, o);
    }
  }
}

// out = a + (y ? dy * [y > 0] : b)   (the gradient arriving at a residual block's input)
__global__ void __launch_bounds__(256) add_kernel(const __nv_bfloat16* __restrict__ a,
                                                  const __nv_bfloat16* __restrict__ b,
                                                  const __nv_bfloat16* __restrict__ y, int64_t n8,
                                                  __nv_bfloat16* __restrict__ out) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n8; i += (int64_t)gridDim.x * blockDim.x) {
    float av[8], bv[8], o[8];
    ld8(a + i * 8, av);
    ld8(b + i * 8, bv);
    if (y) {
      float yv[8];
      ld8(y + i * 8, yv);
#pragma unroll
      for (int q = 0; q < 8; ++q) o[q] = av[q] + (yv[q] > 0.f ? bv[q] : 0.f);
    } else {
#pragma unroll
      for (int q = 0; q < 8; ++q) o[q] = av[q] + bv[q];
    }
    st8(out + i * 8, o);
  }
}

// ---------------------------------------------------------------- stride-2 dX by parity class
// The dX of a stride-2 convolution splits by output parity (a, b) = (y % 2, x % 2): only the taps with
// (a + p - kh) and (b + p - kw) even reach class (a, b), each a stride-1 convolution of dz at row /
// column offsets (a + p - kh) / 2 -- no zero products.  filter_taps_kernel builds a class filter
// [Ci][Tc][Co] (bf16) from the master [Co][T][Ci] (fp32) through a tap map; add_s2_kernel interleaves
// the classes back into the [N][2Hs][2Ws][C] gradient while adding the shortcut's classes.
struct TapMap {
  const float* w;
  __nv_bfloat16* out;
  int Co, T, Ci, Tc;
  int src[9];  // source tap of class tap tc
};
struct TapTable {
  TapMap m[16];
  int n;
};
// block = (32 x 32 tile of (ci, co), class tap tc, filter): read along ci, written along co
__global__ void __launch_bounds__(256) filter_taps_kernel(const __grid_constant__ TapTable tab) {
  __shared__ float tile[32][33];
  const TapMap& m = tab.m[blockIdx.z];
  const int tc = blockIdx.y;
  const int tci = (m.Ci + 31) / 32;
  const int ci0 = (blockIdx.x % tci) * 32, co0 = (blockIdx.x / tci) * 32;
  if (tc >= m.Tc || co0 >= m.Co) return;
  const int tx = threadIdx.x & 31, ty = threadIdx.x >> 5;  // 32 x 8
  for (int k = ty; k < 32; k += 8) {
    const int co = co0 + k, ci = ci0 + tx;
    if (co < m.Co && ci < m.Ci) tile[k][tx] = m.w[((size_t)co * m.T + m.src[tc]) * m.Ci + ci];
  }
  __syncthreads();
  for (int k = ty; k < 32; k += 8) {
    const int ci = ci0 + k, co = co0 + tx;
    if (ci < m.Ci && co < m.Co) m.out[((size_t)ci * m.Tc + tc) * m.Co + co] = __float2bfloat16_rn(tile[tx][k]);
  }
}
struct S2Args {
  const __nv_bfloat16* a[4];  // class (y%2, x%2) = 2a+b of the first gradient, [N][Hs][Ws][C] (null: zero)
  const __nv_bfloat16* b[4];  // the same for the second (the shortcut's dX), null: zero
  __nv_bfloat16* out;         // [N][2Hs][2Ws][C]
  int64_t N;
  int Hs, Ws, lc8;
};
__global__ void __launch_bounds__(256) add_s2_kernel(const __grid_constant__ S2Args g) {
  const int Ho = 2 * g.Hs, Wo = 2 * g.Ws;
  const int64_t n = (g.N * Ho * Wo) << g.lc8;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t pix = i >> g.lc8;
    const int c8 = (int)(i & ((1 << g.lc8) - 1));
    const int64_t img = pix / (Ho * Wo);
    const int r = (int)(pix - img * Ho * Wo), y = r / Wo, x = r - y * Wo;
    const int cls = (y & 1) * 2 + (x & 1);
    const size_t src = ((((size_t)img * g.Hs + (y >> 1)) * g.Ws + (x >> 1)) << g.lc8) * 8 + c8 * 8;
    float va[8] = {0, 0, 0, 0, 0, 0, 0, 0}, vb[8] = {0, 0, 0, 0, 0, 0, 0, 0}, o[8];
    if (g.a[cls]) ld8(g.a[cls] + src, va);
    if (g.b[cls]) ld8(g.b[cls] + src, vb);
#pragma unroll
    for (int q = 0; q < 8; ++q) o[q] = va[q] + vb[q];
    st8(g.out + i * 8, o);
  }
}

// ---------------------------------------------------------------- zero insertion
// up[n][y][x][c] = src[n][y/s][x/s][c] when y and x are multiples of s, else 0 ([N][s*Hs][s*Ws][C]):
// the dX of a stride-s convolution becomes a stride-1 convolution of `up` with the flipped filter
// (the transposed convolution's gather with its zero taps made explicit), so it runs as an implicit GEMM.
__global__ void __launch_bounds__(256) upsample_kernel(const __nv_bfloat16* __restrict__ src, int64_t rows, int Hs,
                                                       int Ws, int lc8, int s, __nv_bfloat16* __restrict__ up) {
  const int Hu = Hs * s, Wu = Ws * s;
  const int64_t n = rows * ((int64_t)Hu * Wu) << lc8;  // 16-byte chunks of up
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t pix = i >> lc8;
    const int c8 = (int)(i & ((1 << lc8) - 1));
    const int64_t img = pix / ((int64_t)Hu * Wu);
    const int r = (int)(pix - img * Hu * Wu), y = r / Wu, x = r - y * Wu;
    uint4 v = make_uint4(0, 0, 0, 0);
    if ((y % s) == 0 && (x % s) == 0)
      v = *(const uint4*)(src + ((((size_t)img * Hs + y / s) * Ws + x / s) << lc8) * 8 + c8 * 8);
    ((uint4*)up)[i] = v;
  }
}

// ---------------------------------------------------------------- head
// Per EST (one block): pooled[n][c] = mean of the 16 positions (4x4) in order; logits = pooled Wfc^T + b
// (c ascending); loss = mean_n CE(softmax(logits), label); dlogits = (p - onehot)/B; per-EST dWfc, dbfc
// (n ascending) into the EST's gradient slot; dx[n][pos][c] = (sum_k dlogits[n][k] Wfc[k][c]) / 16.
constexpr int HEAD_C = 512, HEAD_K = 10, HEAD_POS = 16;
__global__ void __launch_bounds__(512) head_kernel(const __nv_bfloat16* __restrict__ x, const int32_t* __restrict__ labels,
                                                   const float* __restrict__ W, const float* __restrict__ bias, int B,
                                                   float* __restrict__ dW, float* __restrict__ db, int64_t grad_stride,
                                                   float* __restrict__ loss, __nv_bfloat16* __restrict__ dx) {
  extern __shared__ float hsm[];
  float* pooled = hsm;                    // [B][512]
  float* dlog = pooled + B * HEAD_C;      // [B][10]
  const int e = blockIdx.x, t = threadIdx.x;
  const size_t img0 = (size_t)e * B;
  for (int n = 0; n < B; ++n) {  // thread = channel
    float acc = 0.f;
    for (int p = 0; p < HEAD_POS; ++p) acc += __bfloat162float(x[((img0 + n) * HEAD_POS + p) * HEAD_C + t]);
    pooled[n * HEAD_C + t] = acc * (1.f / HEAD_POS);
  }
  __syncthreads();
  for (int i = t; i < B * HEAD_K; i += blockDim.x) {
    const int n = i / HEAD_K, k = i - n * HEAD_K;
    float acc = bias[k];
    for (int c = 0; c < HEAD_C; ++c) acc += pooled[n * HEAD_C + c] * W[k * HEAD_C + c];
    dlog[i] = acc;
  }
  __syncthreads();
  if (t < B) {  // softmax + CE per image
    float* l = dlog + t * HEAD_K;
    float m = l[0];
    for (int k = 1; k < HEAD_K; ++k) m = fmaxf(m, l[k]);
    float s = 0.f;
    for (int k = 0; k < HEAD_K; ++k) s += expf(l[k] - m);
    const int y = labels[img0 + t];
    const float lse = m + logf(s);
    const float ce = lse - l[y];
    for (int k = 0; k < HEAD_K; ++k) l[k] = (expf(l[k] - lse) - (k == y ? 1.f : 0.f)) / (float)B;
    hsm[B * HEAD_C + B * HEAD_K + t] = ce;
  }
  __syncthreads();
  if (t == 0) {
    float acc = 0.f;
    for (int n = 0; n < B; ++n) acc += hsm[B * HEAD_C + B * HEAD_K + n];
    loss[e] = acc / (float)B;
  }
  for (int k = 0; k < HEAD_K; ++k) {  // dW[k][c], thread = c
    float acc = 0.f;
    for (int n = 0; n < B; ++n) acc += dlog[n * HEAD_K + k] * pooled[n * HEAD_C + t];
    dW[(size_t)e * grad_stride + k * HEAD_C + t] = acc;
  }
  if (t < HEAD_K) {
    float acc = 0.f;
    for (int n = 0; n < B; ++n) acc += dlog[n * HEAD_K + t];
    db[(size_t)e * grad_stride + t] = acc;
  }
  for (int n = 0; n < B; ++n) {
    float acc = 0.f;
    for (int k = 0; k < HEAD_K; ++k) acc += dlog[n * HEAD_K + k] * W[k * HEAD_C + t];
    const __nv_bfloat16 g = __float2bfloat16_rn(acc * (1.f / HEAD_POS));
    for (int p = 0; p < HEAD_POS; ++p) dx[((img0 + n) * HEAD_POS + p) * HEAD_C + t] = g;
  }
}

// ---------------------------------------------------------------- weights
// master W [Co][KH*KW][Ci] fp32 -> Wb [Co][KH*KW*Ci] bf16 (forward B operand) and
// Wt [Ci][KH*KW][Co] bf16 (the dX product's B operand; taps reversed when flip), one launch for a table
struct ConvW {
  const float* w;
  __nv_bfloat16* wb;
  __nv_bfloat16* wt;
  int Co, T, Ci;  // T = KH*KW
  int flip;       // wt taps reversed (stride-1 dX as a forward convolution of dz with the flipped filter)
};
constexpr int MAX_CONV = 32;
struct ConvWTable {
  ConvW m[MAX_CONV];
  int n;
};
// block = (32 x 32 tile of (ci, co), tap t, conv): wb written along ci as read; wt through a shared-
// memory transpose, written along co
__global__ void __launch_bounds__(256) conv_weights_kernel(const __grid_constant__ ConvWTable tab) {
  __shared__ float tile[32][33];
  const ConvW& m = tab.m[blockIdx.z];
  const int t = blockIdx.y;
  const int tci = (m.Ci + 31) / 32;
  const int ci0 = (blockIdx.x % tci) * 32, co0 = (blockIdx.x / tci) * 32;
  if (t >= m.T || co0 >= m.Co) return;
  const int tx = threadIdx.x & 31, ty = threadIdx.x >> 5;  // 32 x 8
  for (int k = ty; k < 32; k += 8) {
    const int co = co0 + k, ci = ci0 + tx;
    if (co < m.Co && ci < m.Ci) {
      const size_t i = ((size_t)co * m.T + t) * m.Ci + ci;
      const float v = m.w[i];
      m.wb[i] = __float2bfloat16_rn(v);
      tile[k][tx] = v;
    }
  }
  __syncthreads();
  const int tt = m.flip ? m.T - 1 - t : t;
  for (int k = ty; k < 32; k += 8) {
    const int ci = ci0 + k, co = co0 + tx;
    if (ci < m.Ci && co < m.Co) m.wt[((size_t)ci * m.T + tt) * m.Co + co] = __float2bfloat16_rn(tile[tx][k]);
  }
}

// Weight gradients computed in fixed pixel splits (split-K with a pinned order): out[e] = sum over
// sp ascending of part[e*splits + sp]  (n floats each), written at out + e*out_stride.
__global__ void fold_splits_kernel(const float* __restrict__ part, int E, int splits, int64_t n,
                                   float* __restrict__ out, int64_t out_stride) {
  const int64_t total = (int64_t)E * (n / 4);
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < total; i += (int64_t)gridDim.x * blockDim.x) {
    const int e = (int)(i / (n / 4));
    const int64_t j = (i - (int64_t)e * (n / 4)) * 4;
    const float* p = part + (size_t)e * splits * n + j;
    float4 acc = *(const float4*)p;
    int sp = 1;
    for (; sp + 3 < splits; sp += 4) {  // four loads in flight, added in split order
      float4 v[4];
#pragma unroll
      for (int u = 0; u < 4; ++u) v[u] = *(const float4*)(p + (size_t)(sp + u) * n);
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        acc.x += v[u].x;
        acc.y += v[u].y;
        acc.z += v[u].z;
        acc.w += v[u].w;
      }
    }
    for (; sp < splits; ++sp) {
      const float4 v = *(const float4*)(p + (size_t)sp * n);
      acc.x += v.x;
      acc.y += v.y;
      acc.z += v.z;
      acc.w += v.w;
    }
    *(float4*)(out + (size_t)e * out_stride + j) = acc;
  }
}

}  // namespace cnn

// ----------------------------------------------------------------- launchers
static int ok_or_cuda_c();
static int grid_n(int64_t n);
int cnn_fold_splits_launch(const float* part, int E, int splits, int64_t n, float* out, int64_t out_stride,
                           cudaStream_t s) {
  if (n % 4 || out_stride % 4) return ERR_INPUT;
  cnn::fold_splits_kernel<<<grid_n((int64_t)E * n / 4), 256, 0, s>>>(part, E, splits, n, out, out_stride);
  return ok_or_cuda_c();
}
static int ok_or_cuda_c() { return cudaGetLastError() == cudaSuccess ? OK : ERR_CUDA; }
static int grid_n(int64_t n) {
  const int64_t g = (n + 255) / 256;
  return (int)(g > 148 * 16 ? 148 * 16 : (g < 1 ? 1 : g));
}

int cnn_data_launch(uint64_t seed, const int64_t* cursor, int est_base, int E, int B, void* x, int32_t* labels,
                    cudaStream_t s) {
  cnn::data_kernel<<<grid_n((int64_t)E * B * 1024), 256, 0, s>>>(seed, cursor, est_base, B, E, (__nv_bfloat16*)x,
                                                                 labels);
  return ok_or_cuda_c();
}

int cnn_im2col_launch(const void* src, void* col, int N, int Hs, int Ws, int C, int Ho, int Wo, int KH, int KW,
                      int stride, int pad, int transposed, cudaStream_t s) {
  if (C % 8) return ERR_INPUT;
  const int cg = C / 8;
  if ((int64_t)N * Ho * Wo >= (int64_t)1 << 31 || (cg & (cg - 1)) || KW > 3 || KH > 3 ||
      (stride != 1 && stride != 2))
    return ERR_INPUT;
  int lcg = 0;
  while ((1 << lcg) < cg) ++lcg;
  const cnn::ColArgs a{(const __nv_bfloat16*)src, (__nv_bfloat16*)col, N, Hs, Ws, C, Ho, Wo, KH, KW, stride, pad,
                       transposed};
  const int K8 = KH * KW * cg;
  if (K8 < 32)
    cnn::im2col_kernel<true><<<grid_n((int64_t)N * Ho * Wo * K8), 256, 0, s>>>(a, lcg);
  else
    cnn::im2col_kernel<false><<<grid_n((int64_t)N * Ho * Wo * 32), 256, 0, s>>>(a, lcg);
  return ok_or_cuda_c();
}

// mode 0: mean, rstd, running stats (one pass); mode 2: backward sums (+ dgamma, dbeta)
int cnn_bn_stats_launch(int mode, const void* z, const void* dy, const void* y, float* mean, float* rstd,
                        float* sg, float* sgx, float* part, float* run_mean, float* run_var, int64_t run_stride,
                        float* dgamma, float* dbeta, int64_t grad_stride, int E, int R, int C, float eps,
                        cudaStream_t s) {
  // C in {8, 16, 32, 64} or a multiple of 64 (64-channel slices per block)
  if (!(C == 8 || C == 16 || C == 32 || C % 64 == 0) || C > 2048 || R < 2 || mode == 1) return ERR_INPUT;
  const int chunk = cnn::chunk_rows(C, mode), chunks = (R + chunk - 1) / chunk;
  cnn::StatArgs sa{(const __nv_bfloat16*)z, (const __nv_bfloat16*)dy, (const __nv_bfloat16*)y,
                   mean, rstd, part, C, R, mode, chunk};
  const dim3 grid(chunks, C > 64 ? C / 64 : 1, E);
  if (mode == 0) cnn::stats_kernel<0><<<grid, 256, 0, s>>>(sa);
  else cnn::stats_kernel<2><<<grid, 256, 0, s>>>(sa);
  cnn::FoldArgs fa{};
  fa.part = part;
  fa.out0 = mode == 0 ? mean : sg;
  fa.out1 = mode == 0 ? rstd : sgx;
  fa.z = (const __nv_bfloat16*)z;
  fa.run_mean = run_mean;
  fa.run_var = run_var;
  fa.run_stride = run_stride;
  fa.dgamma = dgamma;
  fa.dbeta = dbeta;
  fa.grad_stride = grad_stride;
  fa.C = C;
  fa.R = R;
  fa.E = E;
  fa.chunks = chunks;
  fa.mode = mode;
  fa.eps = eps;
  cnn::fold_kernel<<<grid_n((int64_t)E * C * 32), 256, 0, s>>>(fa);
  return ok_or_cuda_c();
}

// rows per BatchNorm block: ~4 blocks per SM over the launch, a whole number of unrolled row steps
static int bn_rows_per(int E, int R, int C) {
  const int step = cnn::BN_UNROLL * (cnn::BN_THREADS / (C / 8));
  const int64_t want = ((int64_t)R * E + 4 * 148 - 1) / (4 * 148);
  const int64_t rp = (want + step - 1) / step * step;
  return (int)(rp < R ? rp : R);
}
int cnn_bn_apply_launch(const void* z, const void* res, const float* mean, const float* rstd, const float* gamma,
                        const float* beta, int E, int R, int C, int relu, void* y, cudaStream_t s) {
  if (C % 64 || C > 512 || (int64_t)R * C / 8 >= (int64_t)1 << 31) return ERR_INPUT;
  const int rows_per = bn_rows_per(E, R, C);
  const dim3 grid((R + rows_per - 1) / rows_per, E);
  cnn::bn_apply_kernel<<<grid, cnn::BN_THREADS, 4 * C * sizeof(float), s>>>(
      (const __nv_bfloat16*)z, (const __nv_bfloat16*)res, mean, rstd, gamma, beta, C, R, relu, rows_per,
      (__nv_bfloat16*)y);
  return ok_or_cuda_c();
}

int cnn_bn_bwd_launch(const void* z, const void* dy, const void* y, const float* mean, const float* rstd,
                      const float* sg, const float* sgx, const float* gamma, int E, int R, int C, void* dz,
                      cudaStream_t s) {
  if (C % 64 || C > 512 || (int64_t)R * C / 8 >= (int64_t)1 << 31) return ERR_INPUT;
  const int rows_per = bn_rows_per(E, R, C);
  const dim3 grid((R + rows_per - 1) / rows_per, E);
  cnn::bn_bwd_kernel<<<grid, cnn::BN_THREADS, 5 * C * sizeof(float), s>>>(
      (const __nv_bfloat16*)z, (const __nv_bfloat16*)dy, (const __nv_bfloat16*)y, mean, rstd, sg, sgx, gamma, C, R,
      rows_per, (__nv_bfloat16*)dz);
  return ok_or_cuda_c();
}

int cnn_add_launch(const void* a, const void* b, const void* y, int64_t n, void* out, cudaStream_t s) {
  if (n % 8) return ERR_INPUT;
  cnn::add_kernel<<<grid_n(n / 8), 256, 0, s>>>((const __nv_bfloat16*)a, (const __nv_bfloat16*)b,
                                                (const __nv_bfloat16*)y, n / 8, (__nv_bfloat16*)out);
  return ok_or_cuda_c();
}

int cnn_filter_taps_launch(const float* const* w, void* const* out, const int* Co, const int* T, const int* Ci,
                           const int* Tc, const int* src, int n, cudaStream_t s) {
  if (n < 1 || n > 16) return ERR_INPUT;
  cnn::TapTable tab{};
  int64_t mx = 0;
  for (int i = 0; i < n; ++i) {
    if (Tc[i] < 1 || Tc[i] > 9) return ERR_INPUT;
    cnn::TapMap& m = tab.m[i];
    m.w = w[i];
    m.out = (__nv_bfloat16*)out[i];
    m.Co = Co[i];
    m.T = T[i];
    m.Ci = Ci[i];
    m.Tc = Tc[i];
    for (int t = 0; t < Tc[i]; ++t) {
      if (src[i * 9 + t] < 0 || src[i * 9 + t] >= T[i]) return ERR_INPUT;
      m.src[t] = src[i * 9 + t];
    }
    const int64_t sz = (int64_t)Co[i] * Tc[i] * Ci[i];
    mx = sz > mx ? sz : mx;
  }
  tab.n = n;
  int tiles = 0, tcmax = 0;
  for (int i = 0; i < n; ++i) {
    const int t = ((Ci[i] + 31) / 32) * ((Co[i] + 31) / 32);
    tiles = t > tiles ? t : tiles;
    tcmax = Tc[i] > tcmax ? Tc[i] : tcmax;
  }
  (void)mx;
  cnn::filter_taps_kernel<<<dim3(tiles, tcmax, n), 256, 0, s>>>(tab);
  return ok_or_cuda_c();
}

int cnn_add_s2_launch(const void* const* a, const void* const* b, void* out, int64_t N, int Hs, int Ws, int C,
                      cudaStream_t s) {
  int lc8 = 0;
  while ((8 << lc8) < C) ++lc8;
  if ((8 << lc8) != C) return ERR_INPUT;
  cnn::S2Args g{};
  for (int k = 0; k < 4; ++k) {
    g.a[k] = a ? (const __nv_bfloat16*)a[k] : nullptr;
    g.b[k] = b ? (const __nv_bfloat16*)b[k] : nullptr;
  }
  g.out = (__nv_bfloat16*)out;
  g.N = N;
  g.Hs = Hs;
  g.Ws = Ws;
  g.lc8 = lc8;
  cnn::add_s2_kernel<<<grid_n(N * 4 * Hs * Ws * (C / 8)), 256, 0, s>>>(g);
  return ok_or_cuda_c();
}

int cnn_upsample_launch(const void* src, int64_t N, int Hs, int Ws, int C, int s, void* up, cudaStream_t st) {
  int lc8 = 0;
  while ((8 << lc8) < C) ++lc8;
  if ((8 << lc8) != C || (s != 1 && s != 2)) return ERR_INPUT;
  cnn::upsample_kernel<<<grid_n(N * Hs * Ws * s * s * (C / 8)), 256, 0, st>>>((const __nv_bfloat16*)src, N, Hs, Ws, lc8,
                                                                              s, (__nv_bfloat16*)up);
  return ok_or_cuda_c();
}

int cnn_head_launch(const void* x, const int32_t* labels, const float* W, const float* bias, int E, int B, float* dW,
                    float* db, int64_t grad_stride, float* loss, void* dx, cudaStream_t s) {
  const int smem = (B * cnn::HEAD_C + B * cnn::HEAD_K + B) * (int)sizeof(float);
  static bool attr = false;
  if (!attr) {
    if (cudaFuncSetAttribute(cnn::head_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024) !=
        cudaSuccess)
      return ERR_CUDA;
    attr = true;
  }
  if (B < 1 || smem > 200 * 1024) return ERR_INPUT;
  cnn::head_kernel<<<E, cnn::HEAD_C, smem, s>>>((const __nv_bfloat16*)x, labels, W, bias, B, dW, db, grad_stride, loss,
                                                (__nv_bfloat16*)dx);
  return ok_or_cuda_c();
}

int cnn_conv_weights_launch(const float* const* w, void* const* wb, void* const* wt, const int* Co, const int* T,
                            const int* Ci, const int* flip, int n, cudaStream_t s) {
  if (n < 1 || n > cnn::MAX_CONV) return ERR_INPUT;
  cnn::ConvWTable tab{};
  int64_t mx = 0;
  for (int i = 0; i < n; ++i) {
    tab.m[i] = cnn::ConvW{w[i], (__nv_bfloat16*)wb[i], (__nv_bfloat16*)wt[i], Co[i], T[i], Ci[i], flip ? flip[i] : 0};
    const int64_t sz = (int64_t)Co[i] * T[i] * Ci[i];
    mx = sz > mx ? sz : mx;
  }
  tab.n = n;
  int tiles = 0, tmax = 0;
  for (int i = 0; i < n; ++i) {
    const int tl = ((Ci[i] + 31) / 32) * ((Co[i] + 31) / 32);
    tiles = tl > tiles ? tl : tiles;
    tmax = T[i] > tmax ? T[i] : tmax;
  }
  (void)mx;
  cnn::conv_weights_kernel<<<dim3(tiles, tmax, n), 256, 0, s>>>(tab);
  return ok_or_cuda_c();
}

}  // namespace bt
