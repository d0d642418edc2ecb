// bt_bert.cu -- the kernels between the GEMMs of a per-EST BERT encoder step
// (C4, BASELINE.json configs[3]).  No reference
// implementation exists for this model; the EasyScale contract
// it keeps is the reference's: every random draw is keyed by the EST's global
// rank and the step (counter-form splitmix64, as model.py:151-161 keys dropout
// by rank), and every reduction has a shape fixed by the EST's own data, so
// an EST's gradients are the same bits whichever launch group / GPU runs it.
//
// Layout: the tokens of local EST e are rows [e*Te, (e+1)*Te) of every
// activation matrix; sequence s of the launch is rows [s*128, s*128+128).
//   qkv  [T][3*Dm] bf16  (Q | K | V, head h at columns h*64 of each third)
//   ctx  [T][Dm]   bf16
//   LayerNorm input sums / outputs fp32 [T][Dm], bf16 copies for the GEMMs.
//
// Kernels:
//   attn_fwd / attn_bwd  persistent CTAs walking (sequence, head) items with
//                        cp.async double buffering; 8 warps x 16 query rows,
//                        mma.sync m16n8k16 bf16 (S = QK^T/8, softmax, keyed
//                        dropout, PV); the backward recomputes P from Q, K
//                        (same instructions -> same bits) and sums dV, dK over
//                        query rows in ascending k-steps;
//   ln_fwd               x = resid + dropout(branch + bias); y = LN(x)
//                        (residual stream fp32; GEMM outputs and gradients
//                        between GEMMs bf16, as mixed-precision training keeps them)
//                        (one warp per row, butterfly sums: fixed order);
//   ln_bwd               dx = LN'(dy1 + dy2); branch grad = dropout'(dx);
//                        per-EST gamma/beta/bias column partials over fixed
//                        64-row chunks, folded in chunk order (ln_fold);
//   data / mse           synthetic per-EST inputs / regression head.
#include <cuda_bf16.h>
#include <cuda_runtime.h>
#include <stdint.h>
#include <stdlib.h>

#include "bt_common.cuh"

namespace bt {
namespace bert {

constexpr uint64_t TAG_BERT_X = 0x4245'5254'5f58'4441ull;      // "BERT_XDA"
constexpr uint64_t TAG_BERT_Y = 0x4245'5254'5f59'4441ull;      // "BERT_YDA"
constexpr uint64_t TAG_BERT_HDROP = 0x4245'5254'4844'5250ull;  // "BERTHDRP" hidden dropout
constexpr uint64_t TAG_BERT_ADROP = 0x4245'5254'4144'5250ull;  // "BERTADRP" attention-probability dropout

constexpr int SEQ = 128, HD = 64;
constexpr int AT_WARPS = 8, AT_THREADS = 32 * AT_WARPS;
constexpr int LDS = HD + 8;     // bf16 row stride of Q/K/V/dO tiles (144 B: conflict-free ldmatrix)
constexpr int LDP = SEQ + 8;    // bf16 row stride of the P / dS tiles (272 B)
constexpr int LN_CHUNK = 16;    // rows per ln_bwd partial (fixed: part of the reduction's shape)

__device__ __forceinline__ uint32_t su32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void ldsm_x4(uint32_t addr, uint32_t* r) {
  asm volatile("ldmatrix.sync.aligned.m8n8.x4.shared.b16 {%0,%1,%2,%3}, [%4];"
               : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3])
               : "r"(addr));
}
__device__ __forceinline__ void ldsm_x4_t(uint32_t addr, uint32_t* r) {
  asm volatile("ldmatrix.sync.aligned.m8n8.x4.trans.shared.b16 {%0,%1,%2,%3}, [%4];"
               : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3])
               : "r"(addr));
}
__device__ __forceinline__ void mma16816(float* c, const uint32_t* a, uint32_t b0, uint32_t b1) {
  asm volatile(
      "mma.sync.aligned.m16n8k16.row.col.f32.bf16.bf16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, "
      "{%0,%1,%2,%3};"
      : "+f"(c[0]), "+f"(c[1]), "+f"(c[2]), "+f"(c[3])
      : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b0), "r"(b1));
}
__device__ __forceinline__ uint32_t pack2(float lo, float hi) {
  const __nv_bfloat162 v = __floats2bfloat162_rn(lo, hi);
  return *(const uint32_t*)&v;
}

// [128][64] bf16 tile (row stride `ld` elements in global) -> smem [128][LDS], asynchronously
// (cp.async 16 B; the persistent attention kernels prefetch the next (sequence, head) item's
// tiles while computing the current one)
__device__ __forceinline__ void cp_async16(uint32_t dst, const void* src) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(dst), "l"(src) : "memory");
}
__device__ __forceinline__ void cp_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
__device__ __forceinline__ void cp_wait1() { asm volatile("cp.async.wait_group 1;" ::: "memory"); }
__device__ __forceinline__ void load_tile_async(__nv_bfloat16* dst, const __nv_bfloat16* src, int ld) {
  const uint32_t d = su32(dst);
  for (int c = threadIdx.x; c < SEQ * (HD / 8); c += AT_THREADS) {
    const int r = c >> 3, k = (c & 7) * 8;
    cp_async16(d + 2u * (r * LDS + k), src + (size_t)r * ld + k);
  }
}

// Attention-probability dropout.  One splitmix64 draw per (16-row block, row g < 8, column pair)
// covers 4 units as 16-bit fields: field (hi*2 + lo) is (row 16*r16 + g + 8*hi, column 2*jp + lo);
// a unit is dropped iff its field < ceil(p * 2^16).  Counter of the draw: nb + (r16*8 + g)*64 + jp,
// nb = 4096 draws per (EST, step, layer, sequence, head).  In the mma fragment layout this is one
// draw per thread per 8-column tile, covering the thread's rows g and g+8, columns 2c, 2c+1.
__device__ __forceinline__ uint32_t threshold32(float p) { return p > 0.f ? (uint32_t)ceil((double)p * 0x1p32) : 0u; }
__device__ __forceinline__ uint32_t threshold16(float p) { return p > 0.f ? (uint32_t)ceil((double)p * 65536.0) : 0u; }
__device__ __forceinline__ void attn_mask4(uint64_t sd, uint64_t n, uint32_t thr, float keep, float* m) {
  if (thr == 0) {
    m[0] = m[1] = m[2] = m[3] = 1.f;
    return;
  }
  const uint64_t r = draw_raw(sd, n);
  const uint32_t lo = (uint32_t)r, hi = (uint32_t)(r >> 32);
  m[0] = (lo & 0xFFFFu) < thr ? 0.f : keep;
  m[1] = (lo >> 16) < thr ? 0.f : keep;
  m[2] = (hi & 0xFFFFu) < thr ? 0.f : keep;
  m[3] = (hi >> 16) < thr ? 0.f : keep;
}

// S = softmax(Q_w K^T / 8) for the warp's 16 query rows: s[nt][0..1] = row g, s[nt][2..3] = row g+8,
// columns nt*8 + 2*(lane&3) + {0,1}.  Fixed instruction sequence -> the backward recomputes the same bits.
__device__ __forceinline__ void warp_softmax(const __nv_bfloat16* Qs, const __nv_bfloat16* Ks, int w, int lane,
                                             float (&s)[16][4]) {
#pragma unroll
  for (int nt = 0; nt < 16; ++nt) s[nt][0] = s[nt][1] = s[nt][2] = s[nt][3] = 0.f;
  const uint32_t qb = su32(Qs), kb = su32(Ks);
#pragma unroll
  for (int kk = 0; kk < HD / 16; ++kk) {
    uint32_t a[4];
    ldsm_x4(qb + 2u * ((16 * w + (lane & 7) + ((lane >> 3) & 1) * 8) * LDS + kk * 16 + (lane >> 4) * 8), a);
#pragma unroll
    for (int n2 = 0; n2 < 8; ++n2) {
      uint32_t b[4];
      ldsm_x4(kb + 2u * ((n2 * 16 + (lane & 7) + (lane >> 4) * 8) * LDS + kk * 16 + ((lane >> 3) & 1) * 8), b);
      mma16816(s[2 * n2], a, b[0], b[1]);
      mma16816(s[2 * n2 + 1], a, b[2], b[3]);
    }
  }
  // scores in log2 units: S/8 * log2(e), so exp(S/8 - max) = exp2(s - max2) (ex2.approx)
  constexpr float SC = 0.125f * 1.4426950408889634f;
  float m0 = -INFINITY, m1 = -INFINITY;
#pragma unroll
  for (int nt = 0; nt < 16; ++nt) {
#pragma unroll
    for (int q = 0; q < 4; ++q) s[nt][q] *= SC;
    m0 = fmaxf(m0, fmaxf(s[nt][0], s[nt][1]));
    m1 = fmaxf(m1, fmaxf(s[nt][2], s[nt][3]));
  }
  m0 = fmaxf(m0, __shfl_xor_sync(0xffffffffu, m0, 1));
  m0 = fmaxf(m0, __shfl_xor_sync(0xffffffffu, m0, 2));
  m1 = fmaxf(m1, __shfl_xor_sync(0xffffffffu, m1, 1));
  m1 = fmaxf(m1, __shfl_xor_sync(0xffffffffu, m1, 2));
  float l0 = 0.f, l1 = 0.f;
#pragma unroll
  for (int nt = 0; nt < 16; ++nt) {
    s[nt][0] = exp2f(s[nt][0] - m0);
    l0 += s[nt][0];
    s[nt][1] = exp2f(s[nt][1] - m0);
    l0 += s[nt][1];
    s[nt][2] = exp2f(s[nt][2] - m1);
    l1 += s[nt][2];
    s[nt][3] = exp2f(s[nt][3] - m1);
    l1 += s[nt][3];
  }
  l0 += __shfl_xor_sync(0xffffffffu, l0, 1);  // a+b == b+a: all four lanes of a row agree bitwise
  l0 += __shfl_xor_sync(0xffffffffu, l0, 2);
  l1 += __shfl_xor_sync(0xffffffffu, l1, 1);
  l1 += __shfl_xor_sync(0xffffffffu, l1, 2);
  const float i0 = __frcp_rn(l0), i1 = __frcp_rn(l1);
#pragma unroll
  for (int nt = 0; nt < 16; ++nt) {
    s[nt][0] *= i0;
    s[nt][1] *= i0;
    s[nt][2] *= i1;
    s[nt][3] *= i1;
  }
}

struct AttnArgs {
  const __nv_bfloat16* qkv;  // [T][3*Dm]
  const __nv_bfloat16* dctx; // [T][Dm] (backward)
  __nv_bfloat16* out;        // ctx [T][Dm] (forward) / dqkv [T][3*Dm] (backward)
  int Dm, H, seqs_per_est, est_base, L, layer, n_items;
  uint64_t seed;
  int64_t step;
  float p;
  const int64_t* step_dev;  // when set, the step is read from device memory (CUDA-graph replays)
};
__device__ __forceinline__ int64_t cur_step(int64_t step, const int64_t* step_dev) {
  return step_dev ? *step_dev : step;
}

// counter base of (EST stream, step, layer, sequence-in-EST, head): 4096 draws (16384 units) follow
__device__ __forceinline__ uint64_t attn_counter_base(const AttnArgs& a, int64_t step, int sl, int h) {
  return ((((uint64_t)step * a.L + a.layer) * a.seqs_per_est + sl) * a.H + h) * (uint64_t)(SEQ * SEQ / 4);
}

// Persistent: CTA walks items (sequence s, head h) = (it / H, it % H), it += gridDim.x; the next
// item's tiles stream into the other buffer (cp.async) while this one computes.
constexpr int ATF_BUF = 3 * SEQ * LDS;  // bf16 elements per buffer (Q, K, V)
constexpr int ATF_SMEM = 2 * ATF_BUF * 2;
__global__ void __launch_bounds__(AT_THREADS) attn_fwd_kernel(const AttnArgs a) {
  extern __shared__ __align__(16) uint8_t at_smem[];
  __nv_bfloat16* const buf0 = (__nv_bfloat16*)at_smem;
  const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int ld = 3 * a.Dm;
  const int64_t step = cur_step(a.step, a.step_dev);
  auto issue = [&](int it, __nv_bfloat16* bq) {
    if (it < a.n_items) {
      const __nv_bfloat16* base = a.qkv + (size_t)(it / a.H) * SEQ * ld + (it % a.H) * HD;
      load_tile_async(bq, base, ld);
      load_tile_async(bq + SEQ * LDS, base + a.Dm, ld);
      load_tile_async(bq + 2 * SEQ * LDS, base + 2 * a.Dm, ld);
    }
    cp_commit();
  };
  const uint32_t thr = threshold16(a.p);
  const float keep = a.p < 1.f ? 1.f / (1.f - a.p) : 0.f;
  const int g = lane >> 2, i0 = 16 * w + g, c0 = 2 * (lane & 3);
  int cur = 0;
  issue(blockIdx.x, buf0);
  for (int it = blockIdx.x; it < a.n_items; it += gridDim.x, cur ^= 1) {
    __nv_bfloat16* const Qs = buf0 + cur * ATF_BUF;
    __nv_bfloat16* const Ks = Qs + SEQ * LDS;
    __nv_bfloat16* const Vs = Ks + SEQ * LDS;
    issue(it + gridDim.x, buf0 + (cur ^ 1) * ATF_BUF);
    cp_wait1();
    __syncthreads();
    const int s = it / a.H, h = it % a.H;
    float P[16][4];
    warp_softmax(Qs, Ks, w, lane, P);
    const int e = s / a.seqs_per_est, sl = s - e * a.seqs_per_est;
    const uint64_t sd = derive3(TAG_BERT_ADROP, a.seed, (uint64_t)(a.est_base + e));
    const uint64_t nb = attn_counter_base(a, step, sl, h) + (uint64_t)(w * 8 + g) * 64 + (lane & 3);
    uint32_t pa[8][4];  // dropped P as bf16 A fragments, k-step kv = keys 16kv..16kv+15
#pragma unroll
    for (int nt = 0; nt < 16; ++nt) {
      float m[4];
      attn_mask4(sd, nb + nt * 4, thr, keep, m);
      pa[nt >> 1][(nt & 1) * 2 + 0] = pack2(P[nt][0] * m[0], P[nt][1] * m[1]);
      pa[nt >> 1][(nt & 1) * 2 + 1] = pack2(P[nt][2] * m[2], P[nt][3] * m[3]);
    }
    float o[8][4];
#pragma unroll
    for (int dt = 0; dt < 8; ++dt) o[dt][0] = o[dt][1] = o[dt][2] = o[dt][3] = 0.f;
    const uint32_t vb = su32(Vs);
#pragma unroll
    for (int kv = 0; kv < 8; ++kv) {
#pragma unroll
      for (int d2 = 0; d2 < 4; ++d2) {
        uint32_t b[4];
        ldsm_x4_t(vb + 2u * ((kv * 16 + (lane & 7) + ((lane >> 3) & 1) * 8) * LDS + d2 * 16 + (lane >> 4) * 8), b);
        mma16816(o[2 * d2], pa[kv], b[0], b[1]);
        mma16816(o[2 * d2 + 1], pa[kv], b[2], b[3]);
      }
    }
    __nv_bfloat16* out = a.out + (size_t)s * SEQ * a.Dm + h * HD;
#pragma unroll
    for (int dt = 0; dt < 8; ++dt) {
      *(uint32_t*)(out + (size_t)i0 * a.Dm + dt * 8 + c0) = pack2(o[dt][0], o[dt][1]);
      *(uint32_t*)(out + (size_t)(i0 + 8) * a.Dm + dt * 8 + c0) = pack2(o[dt][2], o[dt][3]);
    }
    __syncthreads();  // all warps are done with this buffer before it is refilled
  }
}

// dV = Pd^T dO, dP = (dO V^T) * mask, dS = P * (dP - rowsum(dP * P)) / 8, dQ = dS K, dK = dS^T Q
constexpr int ATB_BUF = 4 * SEQ * LDS;  // Q, K, V, dO
constexpr int ATB_SMEM = (2 * ATB_BUF + 2 * SEQ * LDP) * 2;
__global__ void __launch_bounds__(AT_THREADS) attn_bwd_kernel(const AttnArgs a) {
  extern __shared__ __align__(16) uint8_t at_smem[];
  __nv_bfloat16* const buf0 = (__nv_bfloat16*)at_smem;
  __nv_bfloat16* const Ps = buf0 + 2 * ATB_BUF;  // dropped P  [query][key]
  __nv_bfloat16* const dSs = Ps + SEQ * LDP;     // dS / 8     [query][key]
  const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int ld = 3 * a.Dm;
  const int64_t step = cur_step(a.step, a.step_dev);
  auto issue = [&](int it, __nv_bfloat16* bq) {
    if (it < a.n_items) {
      const int s = it / a.H, h = it % a.H;
      const __nv_bfloat16* base = a.qkv + (size_t)s * SEQ * ld + h * HD;
      load_tile_async(bq, base, ld);
      load_tile_async(bq + SEQ * LDS, base + a.Dm, ld);
      load_tile_async(bq + 2 * SEQ * LDS, base + 2 * a.Dm, ld);
      load_tile_async(bq + 3 * SEQ * LDS, a.dctx + (size_t)s * SEQ * a.Dm + h * HD, a.Dm);
    }
    cp_commit();
  };
  const uint32_t thr = threshold16(a.p);
  const float keep = a.p < 1.f ? 1.f / (1.f - a.p) : 0.f;
  const int g = lane >> 2, i0 = 16 * w + g, c0 = 2 * (lane & 3);
  int cur = 0;
  issue(blockIdx.x, buf0);
  for (int it = blockIdx.x; it < a.n_items; it += gridDim.x, cur ^= 1) {
    __nv_bfloat16* const Qs = buf0 + cur * ATB_BUF;
    __nv_bfloat16* const Ks = Qs + SEQ * LDS;
    __nv_bfloat16* const Vs = Ks + SEQ * LDS;
    __nv_bfloat16* const dOs = Vs + SEQ * LDS;
    issue(it + gridDim.x, buf0 + (cur ^ 1) * ATB_BUF);
    cp_wait1();
    __syncthreads();
    const int s = it / a.H, h = it % a.H;
    float P[16][4];
    warp_softmax(Qs, Ks, w, lane, P);
    float dp[16][4];  // dO_w V^T
#pragma unroll
    for (int nt = 0; nt < 16; ++nt) dp[nt][0] = dp[nt][1] = dp[nt][2] = dp[nt][3] = 0.f;
    {
      const uint32_t ob = su32(dOs), vb = su32(Vs);
#pragma unroll
      for (int kk = 0; kk < HD / 16; ++kk) {
        uint32_t af[4];
        ldsm_x4(ob + 2u * ((16 * w + (lane & 7) + ((lane >> 3) & 1) * 8) * LDS + kk * 16 + (lane >> 4) * 8), af);
#pragma unroll
        for (int n2 = 0; n2 < 8; ++n2) {
          uint32_t b[4];
          ldsm_x4(vb + 2u * ((n2 * 16 + (lane & 7) + (lane >> 4) * 8) * LDS + kk * 16 + ((lane >> 3) & 1) * 8), b);
          mma16816(dp[2 * n2], af, b[0], b[1]);
          mma16816(dp[2 * n2 + 1], af, b[2], b[3]);
        }
      }
    }
    const int e = s / a.seqs_per_est, sl = s - e * a.seqs_per_est;
    const uint64_t sd = derive3(TAG_BERT_ADROP, a.seed, (uint64_t)(a.est_base + e));
    const uint64_t nb = attn_counter_base(a, step, sl, h) + (uint64_t)(w * 8 + g) * 64 + (lane & 3);
    float r0 = 0.f, r1 = 0.f;  // rowsum(dP * P), rows i0 / i0+8
#pragma unroll
    for (int nt = 0; nt < 16; ++nt) {
      float m[4];
      attn_mask4(sd, nb + nt * 4, thr, keep, m);
      const int j = nt * 8 + c0;
      *(uint32_t*)(Ps + i0 * LDP + j) = pack2(P[nt][0] * m[0], P[nt][1] * m[1]);
      *(uint32_t*)(Ps + (i0 + 8) * LDP + j) = pack2(P[nt][2] * m[2], P[nt][3] * m[3]);
#pragma unroll
      for (int q = 0; q < 4; ++q) dp[nt][q] *= m[q];
      r0 += dp[nt][0] * P[nt][0];
      r0 += dp[nt][1] * P[nt][1];
      r1 += dp[nt][2] * P[nt][2];
      r1 += dp[nt][3] * P[nt][3];
    }
    r0 += __shfl_xor_sync(0xffffffffu, r0, 1);
    r0 += __shfl_xor_sync(0xffffffffu, r0, 2);
    r1 += __shfl_xor_sync(0xffffffffu, r1, 1);
    r1 += __shfl_xor_sync(0xffffffffu, r1, 2);
    uint32_t da[8][4];  // dS/8 as bf16 A fragments (rows of this warp)
#pragma unroll
    for (int nt = 0; nt < 16; ++nt) {
      const float d0 = P[nt][0] * (dp[nt][0] - r0) * 0.125f, d1 = P[nt][1] * (dp[nt][1] - r0) * 0.125f;
      const float d2 = P[nt][2] * (dp[nt][2] - r1) * 0.125f, d3 = P[nt][3] * (dp[nt][3] - r1) * 0.125f;
      const uint32_t lo = pack2(d0, d1), hi = pack2(d2, d3);
      da[nt >> 1][(nt & 1) * 2 + 0] = lo;
      da[nt >> 1][(nt & 1) * 2 + 1] = hi;
      const int j = nt * 8 + c0;
      *(uint32_t*)(dSs + i0 * LDP + j) = lo;
      *(uint32_t*)(dSs + (i0 + 8) * LDP + j) = hi;
    }
    __nv_bfloat16* dq = a.out + (size_t)s * SEQ * ld + h * HD;
    {  // dQ_w = dS_w K
      float acc[8][4];
#pragma unroll
      for (int dt = 0; dt < 8; ++dt) acc[dt][0] = acc[dt][1] = acc[dt][2] = acc[dt][3] = 0.f;
      const uint32_t kb = su32(Ks);
#pragma unroll
      for (int kv = 0; kv < 8; ++kv) {
#pragma unroll
        for (int d2 = 0; d2 < 4; ++d2) {
          uint32_t b[4];
          ldsm_x4_t(kb + 2u * ((kv * 16 + (lane & 7) + ((lane >> 3) & 1) * 8) * LDS + d2 * 16 + (lane >> 4) * 8), b);
          mma16816(acc[2 * d2], da[kv], b[0], b[1]);
          mma16816(acc[2 * d2 + 1], da[kv], b[2], b[3]);
        }
      }
#pragma unroll
      for (int dt = 0; dt < 8; ++dt) {
        *(uint32_t*)(dq + (size_t)i0 * ld + dt * 8 + c0) = pack2(acc[dt][0], acc[dt][1]);
        *(uint32_t*)(dq + (size_t)(i0 + 8) * ld + dt * 8 + c0) = pack2(acc[dt][2], acc[dt][3]);
      }
    }
    __syncthreads();
    // warp w: key rows 16w..16w+15.  dV = Pd^T dO, dK = dS^T Q; k-steps = ascending query blocks
#pragma unroll 1
    for (int which = 0; which < 2; ++which) {
      const uint32_t ab = su32(which == 0 ? Ps : dSs), bb = su32(which == 0 ? dOs : Qs);
      float acc[8][4];
#pragma unroll
      for (int dt = 0; dt < 8; ++dt) acc[dt][0] = acc[dt][1] = acc[dt][2] = acc[dt][3] = 0.f;
#pragma unroll
      for (int kq = 0; kq < 8; ++kq) {
        uint32_t af[4];
        ldsm_x4_t(ab + 2u * ((kq * 16 + (lane & 7) + (lane >> 4) * 8) * LDP + 16 * w + ((lane >> 3) & 1) * 8), af);
#pragma unroll
        for (int d2 = 0; d2 < 4; ++d2) {
          uint32_t b[4];
          ldsm_x4_t(bb + 2u * ((kq * 16 + (lane & 7) + ((lane >> 3) & 1) * 8) * LDS + d2 * 16 + (lane >> 4) * 8), b);
          mma16816(acc[2 * d2], af, b[0], b[1]);
          mma16816(acc[2 * d2 + 1], af, b[2], b[3]);
        }
      }
      __nv_bfloat16* dst = dq + (which == 0 ? 2 : 1) * a.Dm;
#pragma unroll
      for (int dt = 0; dt < 8; ++dt) {
        *(uint32_t*)(dst + (size_t)i0 * ld + dt * 8 + c0) = pack2(acc[dt][0], acc[dt][1]);
        *(uint32_t*)(dst + (size_t)(i0 + 8) * ld + dt * 8 + c0) = pack2(acc[dt][2], acc[dt][3]);
      }
    }
    __syncthreads();  // Ps / dSs / this buffer free before the next item
  }
}

// ------------------------------------------------------------ LayerNorm
struct LnArgs {
  const float* resid;         // fwd: residual input [T][D] fp32     bwd: dy2 (residual-path grad) fp32 or null
  const __nv_bfloat16* bin;  // fwd: branch GEMM output (no bias)   bwd: dy1 (branch-path grad), both bf16
  const float* bias;    // fwd: branch bias [D]
  const float* gamma;
  const float* beta;
  float* xsum;          // fwd: out, the LN input (kept for backward)   bwd: in
  const float2* stats_in;
  float2* stats;        // fwd: out (mean, rstd) per row
  float* y32;           // fwd: LN output fp32       bwd: dx (LN-input gradient, the residual path)
  __nv_bfloat16* yb;    // fwd: LN output bf16       bwd: dropout'(dx) bf16 (the branch gradient)
  float* part;          // bwd: [E][chunks][3][D] column partials (dgamma, dbeta, dbias)
  // fwd, when rx is set: the residual is the previous LayerNorm's output recomputed from its input rx,
  // statistics rst and affine rg / rb -- the same expression that produced its y32, hence the same bits
  // (-fmad=false) -- so that LayerNorm need not write y32
  const float* rx;
  const float2* rst;
  const float* rg;
  const float* rb;
  int D, Te, rows, est_base, L, layer, site;
  uint64_t seed;
  int64_t step;
  float p, eps;
  const int64_t* step_dev;  // when set, the step is read from device memory (CUDA-graph replays)
};

// Hidden dropout: one splitmix64 draw per 4 consecutive units (16-bit fields, field k = bits [16k, 16k+16)
// decides unit 4q + k; dropped iff field < ceil(p * 2^16)), keyed by (EST stream, step, layer, site, token,
// unit quad).  The forward and the backward regenerate the same masks.
__device__ __forceinline__ void ln_mask4(uint64_t sd, uint64_t n, uint32_t thr, float keep, float* m) {
  if (thr == 0) {
    m[0] = m[1] = m[2] = m[3] = 1.f;
    return;
  }
  const uint64_t r = draw_raw(sd, n >> 2);
#pragma unroll
  for (int k = 0; k < 4; ++k) m[k] = ((uint32_t)(r >> (16 * k)) & 0xFFFFu) < thr ? 0.f : keep;
}
__device__ __forceinline__ uint64_t ln_counter(const LnArgs& a, int64_t step, int tl) {  // element counter of (tl, 0)
  return ((((uint64_t)step * a.L + a.layer) * 2 + a.site) * a.Te + tl) * (uint64_t)a.D;
}
__device__ __forceinline__ float warp_sum(float v) {  // butterfly: every lane ends with the same bits
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}
__device__ __forceinline__ void cp_async8(uint32_t dst, const void* src) {
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" ::"r"(dst), "l"(src) : "memory");
}
__device__ __forceinline__ void cp_wait0() { asm volatile("cp.async.wait_group 0;" ::: "memory"); }

// Packed fp32 pairs (sm_100a FADD2 / FMUL2 / FFMA2).  ptxas contracts a packed product feeding a packed
// addition into FFMA2 even when both are .rn, so every product that feeds an addition is written as an
// explicit fma: the rounding is then the same wherever the expression appears (the residual recompute of
// ln_fwd must reproduce the previous LayerNorm's output bit for bit).
typedef unsigned long long f2;
__device__ __forceinline__ f2 pk(float a, float b) {
  f2 r;
  asm("mov.b64 %0, {%1, %2};" : "=l"(r) : "f"(a), "f"(b));
  return r;
}
__device__ __forceinline__ float2 upk(f2 r) {
  float2 f;
  asm("mov.b64 {%0, %1}, %2;" : "=f"(f.x), "=f"(f.y) : "l"(r));
  return f;
}
__device__ __forceinline__ f2 add2(f2 a, f2 b) {
  f2 r;
  asm("add.rn.f32x2 %0, %1, %2;" : "=l"(r) : "l"(a), "l"(b));
  return r;
}
__device__ __forceinline__ f2 sub2(f2 a, f2 b) {
  f2 r;
  asm("sub.rn.f32x2 %0, %1, %2;" : "=l"(r) : "l"(a), "l"(b));
  return r;
}
__device__ __forceinline__ f2 mul2(f2 a, f2 b) {
  f2 r;
  asm("mul.rn.f32x2 %0, %1, %2;" : "=l"(r) : "l"(a), "l"(b));
  return r;
}
__device__ __forceinline__ f2 fma2(f2 a, f2 b, f2 c) {
  f2 r;
  asm("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(r) : "l"(a), "l"(b), "l"(c));
  return r;
}
// 4 consecutive floats as two pairs
struct f4p { f2 lo, hi; };
__device__ __forceinline__ f4p ld4f(const void* p) {
  const float4 v = *(const float4*)p;
  return {pk(v.x, v.y), pk(v.z, v.w)};
}
__device__ __forceinline__ f4p ld4b(const void* p) {  // 4 bf16
  const uint2 u = *(const uint2*)p;
  const float2 a = __bfloat1622float2(*(const __nv_bfloat162*)&u.x), b = __bfloat1622float2(*(const __nv_bfloat162*)&u.y);
  return {pk(a.x, a.y), pk(b.x, b.y)};
}
__device__ __forceinline__ void st4f(float* p, f4p v) {
  const float2 a = upk(v.lo), b = upk(v.hi);
  *(float4*)p = make_float4(a.x, a.y, b.x, b.y);
}
__device__ __forceinline__ void st4b(__nv_bfloat16* p, f4p v) {
  const float2 a = upk(v.lo), b = upk(v.hi);
  *(uint2*)p = make_uint2(pack2(a.x, a.y), pack2(b.x, b.y));
}
// the LayerNorm output y = ((x - mean) * rstd) * gamma + beta (one rounding per product, then an fma)
__device__ __forceinline__ f2 ln_out(f2 x, f2 mean, f2 rstd, f2 g, f2 b) { return fma2(mul2(sub2(x, mean), rstd), g, b); }

// Lane columns: a row of D = 256 NC is G = 2 NC groups of 4 columns; group g of lane l is columns
// (g >> 1) * 256 + (g & 1) * 128 + 4 l -- 16-byte fp32 / 8-byte bf16 pieces, consecutive across lanes
// (coalesced loads, conflict-free shared-memory reads).
template <int NC>
__device__ __forceinline__ int lcol(int g, int lane) { return (g >> 1) * 256 + (g & 1) * 128 + 4 * lane; }

// Rows stream through a two-slot shared-memory ring per warp (cp.async): each lane copies exactly the pieces
// it later reads, so a lane waits only on its own copies (no warp synchronisation), and the next row's
// bytes are in flight while this row computes.

// ---- forward: x = resid + dropout(branch + bias); y = LN(x).  Persistent blocks (grid-stride over rows,
// one row per warp at a time); bias, gamma, beta (and the previous LayerNorm's gamma / beta when the
// residual is recomputed from its input rx and statistics rst) staged in shared memory once per block.
constexpr int LNF_WARPS = 6;
template <int NC>
struct LnfSlot {
  static constexpr int D = 256 * NC, R = 0, B = D * 4, ST = B + D * 2, BYTES = ST + 256;
  static constexpr int PAR = 5 * D * 4;  // bias, gamma, beta, rg, rb
};
template <int NC>
__global__ void __launch_bounds__(32 * LNF_WARPS) ln_fwd_kernel(const LnArgs a) {
  using S = LnfSlot<NC>;
  constexpr int D = S::D, G = 2 * NC;
  extern __shared__ __align__(16) uint8_t lsm[];
  float* const par = (float*)lsm;  // [5][D]
  const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
  uint8_t* const wr = lsm + S::PAR + (size_t)w * 2 * S::BYTES;
  const int gw = blockIdx.x * LNF_WARPS + w, nw = gridDim.x * LNF_WARPS;
  const bool rc = a.rx != nullptr;
  const float* const rsrc = rc ? a.rx : a.resid;
  auto issue = [&](int t, int slot) {  // 16-byte pieces, L2 only (.cg); the lanes read each other's pieces
    const uint32_t sb = su32(wr + slot * S::BYTES);
#pragma unroll
    for (int k = lane; k < D / 4; k += 32) cp_async16(sb + S::R + k * 16, rsrc + (size_t)t * D + 4 * k);
#pragma unroll
    for (int k = lane; k < D / 8; k += 32) cp_async16(sb + S::B + k * 16, a.bin + (size_t)t * D + 8 * k);
    if (rc && lane == 0) cp_async8(sb + S::ST, a.rst + t);
    cp_commit();
  };
  if (gw < a.rows) issue(gw, 0);
  if (gw + nw < a.rows) issue(gw + nw, 1);
  const float* srcs[5] = {a.bias, a.gamma, a.beta, a.rg, a.rb};
#pragma unroll
  for (int q = 0; q < 5; ++q)
    if (q < 3 || rc)
      for (int i = threadIdx.x * 4; i < D; i += 32 * LNF_WARPS * 4) *(float4*)(par + q * D + i) = *(const float4*)(srcs[q] + i);
  __syncthreads();
  const uint32_t thr = threshold16(a.p);
  const int64_t step = cur_step(a.step, a.step_dev);
  const float keep = a.p < 1.f ? 1.f / (1.f - a.p) : 0.f;
  int n = 0;
  for (int t = gw; t < a.rows; t += nw, ++n) {
    if (t + nw < a.rows) cp_wait1(); else cp_wait0();
    __syncwarp();
    const uint8_t* const sl = wr + (n & 1) * S::BYTES;
    const int e = t / a.Te, tl = t - e * a.Te;
    const uint64_t sd = derive3(TAG_BERT_HDROP, a.seed, (uint64_t)(a.est_base + e));
    const uint64_t n0 = ln_counter(a, step, tl);
    f2 rm = 0, rs = 0;
    if (rc) {
      const float2 q = *(const float2*)(sl + S::ST);
      rm = pk(q.x, q.x);
      rs = pk(q.y, q.y);
    }
    f4p x[G];
    f2 sum = pk(0.f, 0.f);
#pragma unroll
    for (int g = 0; g < G; ++g) {
      const int c = lcol<NC>(g, lane);
      f4p r = ld4f(sl + S::R + c * 4);
      if (rc) {
        const f4p rg = ld4f(par + 3 * D + c), rb = ld4f(par + 4 * D + c);
        r.lo = ln_out(r.lo, rm, rs, rg.lo, rb.lo);
        r.hi = ln_out(r.hi, rm, rs, rg.hi, rb.hi);
      }
      const f4p b = ld4b(sl + S::B + c * 2), bi = ld4f(par + c);
      float m[4];
      ln_mask4(sd, n0 + c, thr, keep, m);
      x[g].lo = fma2(add2(b.lo, bi.lo), pk(m[0], m[1]), r.lo);
      x[g].hi = fma2(add2(b.hi, bi.hi), pk(m[2], m[3]), r.hi);
      sum = add2(sum, add2(x[g].lo, x[g].hi));
    }
    __syncwarp();  // every lane has read the slot
    if (t + 2 * nw < a.rows) issue(t + 2 * nw, n & 1);
    const float2 sf = upk(sum);
    const float mean = warp_sum(sf.x + sf.y) / (float)D;
    const f2 mm = pk(mean, mean);
    f2 sq = pk(0.f, 0.f);
#pragma unroll
    for (int g = 0; g < G; ++g) {
      const f2 d0 = sub2(x[g].lo, mm), d1 = sub2(x[g].hi, mm);
      sq = fma2(d0, d0, sq);
      sq = fma2(d1, d1, sq);
    }
    const float2 qf = upk(sq);
    const float rstd = 1.f / sqrtf(warp_sum(qf.x + qf.y) / (float)D + a.eps);
    const f2 rr = pk(rstd, rstd);
#pragma unroll
    for (int g = 0; g < G; ++g) {
      const int c = lcol<NC>(g, lane);
      const f4p gm = ld4f(par + D + c), bt = ld4f(par + 2 * D + c);
      const f4p y{ln_out(x[g].lo, mm, rr, gm.lo, bt.lo), ln_out(x[g].hi, mm, rr, gm.hi, bt.hi)};
      st4f(a.xsum + (size_t)t * D + c, x[g]);
      if (a.y32) st4f(a.y32 + (size_t)t * D + c, y);
      st4b(a.yb + (size_t)t * D + c, y);
    }
    if (lane == 0) a.stats[t] = make_float2(mean, rstd);
  }
}

// ---- backward: dx = LN'(dy1 + dy2); branch gradient = dropout'(dx); per-chunk column partials.
// Block = one 16-row chunk (LN_CHUNK, fixed: part of the reduction's shape), 4 warps; warp w takes rows
// w, w+4, w+8, w+12 of the chunk in order, accumulating its dgamma / dbeta / dbias partials in registers,
// then the 4 warps' partials are folded in warp order into part[chunk][3][D].
constexpr int LNB_WARPS = 4;
template <int NC, bool DY2>
struct LnbSlot {
  static constexpr int D = 256 * NC, Y1 = 0, Y2 = D * 2, X = Y2 + (DY2 ? D * 4 : 0), ST = X + D * 4, BYTES = ST + 256;
};
template <int NC, bool DY2>
__global__ void __launch_bounds__(32 * LNB_WARPS, 3) ln_bwd_kernel(const LnArgs a) {
  using S = LnbSlot<NC, DY2>;
  constexpr int D = S::D, G = 2 * NC, RPW = LN_CHUNK / LNB_WARPS;
  static_assert(2 * S::BYTES >= 3 * D * 4, "the ring holds the warp's partials at the end");
  extern __shared__ __align__(16) uint8_t lsm[];
  float* const gam = (float*)lsm;
  const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
  uint8_t* const wr = lsm + D * 4 + (size_t)w * 2 * S::BYTES;
  const size_t row0 = (size_t)blockIdx.x * LN_CHUNK;
  const int e = (int)(row0 / (size_t)a.Te), tl0 = (int)(row0 - (size_t)e * a.Te);
  auto issue = [&](int i) {  // row w + 4 i of the chunk into slot i & 1 (16-byte pieces, L2 only)
    const size_t t = row0 + w + LNB_WARPS * i;
    const uint32_t sb = su32(wr + (i & 1) * S::BYTES);
#pragma unroll
    for (int k = lane; k < D / 8; k += 32) cp_async16(sb + S::Y1 + k * 16, a.bin + t * D + 8 * k);
#pragma unroll
    for (int k = lane; k < D / 4; k += 32) {
      if (DY2) cp_async16(sb + S::Y2 + k * 16, a.resid + t * D + 4 * k);
      cp_async16(sb + S::X + k * 16, a.xsum + t * D + 4 * k);
    }
    if (lane == 0) cp_async8(sb + S::ST, a.stats_in + t);
    cp_commit();
  };
  issue(0);
  issue(1);
  for (int i = threadIdx.x * 4; i < D; i += 32 * LNB_WARPS * 4) *(float4*)(gam + i) = *(const float4*)(a.gamma + i);
  __syncthreads();
  const uint64_t sd = derive3(TAG_BERT_HDROP, a.seed, (uint64_t)(a.est_base + e));
  const uint32_t thr = threshold16(a.p);
  const int64_t step = cur_step(a.step, a.step_dev);
  const float keep = a.p < 1.f ? 1.f / (1.f - a.p) : 0.f;
  f4p pg[G], pb[G], pr[G];
#pragma unroll
  for (int g = 0; g < G; ++g) pg[g] = pb[g] = pr[g] = f4p{pk(0.f, 0.f), pk(0.f, 0.f)};
  auto dy_x = [&](const uint8_t* sl, int c, f4p& dy, f4p& xh, f4p& gg, f2 mean, f2 rstd) {
    dy = ld4b(sl + S::Y1 + c * 2);
    if (DY2) {
      const f4p d2 = ld4f(sl + S::Y2 + c * 4);
      dy.lo = add2(dy.lo, d2.lo);
      dy.hi = add2(dy.hi, d2.hi);
    }
    const f4p x = ld4f(sl + S::X + c * 4), gm = ld4f(gam + c);
    xh.lo = mul2(sub2(x.lo, mean), rstd);
    xh.hi = mul2(sub2(x.hi, mean), rstd);
    gg.lo = mul2(dy.lo, gm.lo);
    gg.hi = mul2(dy.hi, gm.hi);
  };
#pragma unroll 1
  for (int i = 0; i < RPW; ++i) {
    if (i + 1 < RPW) cp_wait1(); else cp_wait0();
    __syncwarp();  // the lanes' copies of this row are visible to the warp
    const uint8_t* const sl = wr + (i & 1) * S::BYTES;
    const float2 st = *(const float2*)(sl + S::ST);
    const f2 mean = pk(st.x, st.x), rstd = pk(st.y, st.y);
    const int tl = tl0 + w + LNB_WARPS * i;
    const size_t t = row0 + w + LNB_WARPS * i;
    f2 s1 = pk(0.f, 0.f), s2 = pk(0.f, 0.f);
#pragma unroll
    for (int g = 0; g < G; ++g) {
      f4p dy, xh, gg;
      dy_x(sl, lcol<NC>(g, lane), dy, xh, gg, mean, rstd);
      s1 = add2(s1, add2(gg.lo, gg.hi));
      s2 = fma2(gg.lo, xh.lo, s2);
      s2 = fma2(gg.hi, xh.hi, s2);
    }
    const float2 a1 = upk(s1), a2 = upk(s2);
    const float m1 = warp_sum(a1.x + a1.y) / (float)D, m2 = warp_sum(a2.x + a2.y) / (float)D;
    const f2 M1 = pk(m1, m1), NM2 = pk(-m2, -m2);
    const uint64_t n0 = ln_counter(a, step, tl);
#pragma unroll
    for (int g = 0; g < G; ++g) {
      const int c = lcol<NC>(g, lane);
      f4p dy, xh, gg;
      dy_x(sl, c, dy, xh, gg, mean, rstd);
      f4p dx;  // (gg - m1 - xh m2) rstd
      dx.lo = mul2(fma2(xh.lo, NM2, sub2(gg.lo, M1)), rstd);
      dx.hi = mul2(fma2(xh.hi, NM2, sub2(gg.hi, M1)), rstd);
      st4f(a.y32 + t * D + c, dx);
      float m[4];
      ln_mask4(sd, n0 + c, thr, keep, m);
      const f2 mlo = pk(m[0], m[1]), mhi = pk(m[2], m[3]);
      st4b(a.yb + t * D + c, f4p{mul2(dx.lo, mlo), mul2(dx.hi, mhi)});
      pg[g].lo = fma2(dy.lo, xh.lo, pg[g].lo);
      pg[g].hi = fma2(dy.hi, xh.hi, pg[g].hi);
      pb[g].lo = add2(pb[g].lo, dy.lo);
      pb[g].hi = add2(pb[g].hi, dy.hi);
      pr[g].lo = fma2(dx.lo, mlo, pr[g].lo);
      pr[g].hi = fma2(dx.hi, mhi, pr[g].hi);
    }
    __syncwarp();  // every lane has read the slot
    if (i + 2 < RPW) issue(i + 2);
  }
  // this warp's partials into its (now idle) ring, then the warps folded in order
  float* const pw = (float*)wr;
#pragma unroll
  for (int g = 0; g < G; ++g) {
    const int c = lcol<NC>(g, lane);
    st4f(pw + c, pg[g]);
    st4f(pw + D + c, pb[g]);
    st4f(pw + 2 * D + c, pr[g]);
  }
  __syncthreads();
  float* const out = a.part + (size_t)blockIdx.x * 3 * D;
  for (int i = threadIdx.x * 4; i < 3 * D; i += 32 * LNB_WARPS * 4) {
    f4p acc = ld4f(lsm + D * 4 + i * 4);
#pragma unroll
    for (int ww = 1; ww < LNB_WARPS; ++ww) {
      const f4p v = ld4f(lsm + D * 4 + (size_t)ww * 2 * S::BYTES + i * 4);
      acc.lo = add2(acc.lo, v.lo);
      acc.hi = add2(acc.hi, v.hi);
    }
    st4f(out + i, acc);
  }
}

// per-leaf dgamma / dbeta / dbias = the chunk partials summed in a fixed association: LNF_SEGS segments of
// consecutive chunks, each summed in order by one thread (4 columns, 16-byte loads, 8 in flight), then the
// segments in order.  Block = (leaf, 128 of the 3D columns), threads (segment, column quad).
constexpr int LNF_SEGS = 16;
__global__ void __launch_bounds__(32 * LNF_SEGS) ln_fold_kernel(const float* __restrict__ part, int chunks, int D,
                                                                float* out_g, float* out_b, float* out_r,
                                                                int64_t est_stride) {
  __shared__ float4 seg[LNF_SEGS][32];
  const int e = blockIdx.y, q = threadIdx.x & 31, sg = threadIdx.x >> 5, r = blockIdx.x * 128 + 4 * q;
  const int per = (chunks + LNF_SEGS - 1) / LNF_SEGS, k0 = sg * per, k1 = min(chunks, k0 + per);
  f4p acc{pk(0.f, 0.f), pk(0.f, 0.f)};
  if (r < 3 * D && k0 < k1) {
    const size_t ld = (size_t)3 * D;
    const float* p = part + ((size_t)e * chunks + k0) * ld + r;
    acc = ld4f(p);
    int k = k0 + 1;
    for (; k + 8 <= k1; k += 8) {  // 8 loads in flight, added in order
      float4 v[8];
#pragma unroll
      for (int j = 0; j < 8; ++j) v[j] = __ldg((const float4*)(p + (size_t)(k - k0 + j) * ld));
#pragma unroll
      for (int j = 0; j < 8; ++j) {
        acc.lo = add2(acc.lo, pk(v[j].x, v[j].y));
        acc.hi = add2(acc.hi, pk(v[j].z, v[j].w));
      }
    }
    for (; k < k1; ++k) {
      const f4p v = ld4f(p + (size_t)(k - k0) * ld);
      acc.lo = add2(acc.lo, v.lo);
      acc.hi = add2(acc.hi, v.hi);
    }
  }
  const float2 lo = upk(acc.lo), hi = upk(acc.hi);
  seg[sg][q] = make_float4(lo.x, lo.y, hi.x, hi.y);
  __syncthreads();
  if (sg == 0 && r < 3 * D) {
    f4p v = ld4f(&seg[0][q]);
    for (int z = 1; z < LNF_SEGS; ++z)
      if (z * per < chunks) {
        const f4p u = ld4f(&seg[z][q]);
        v.lo = add2(v.lo, u.lo);
        v.hi = add2(v.hi, u.hi);
      }
    const int which = r / D, c = r - which * D;  // D % 128 == 0: a quad never straddles gamma / beta / bias
    float* dst = which == 0 ? out_g : (which == 1 ? out_b : out_r);
    st4f(dst + (size_t)e * est_stride + c, v);
  }
}

// ------------------------------------------------------------ data / head
__device__ __forceinline__ void st8(float* p, const float* v) {
  *(float4*)p = make_float4(v[0], v[1], v[2], v[3]);
  *(float4*)(p + 4) = make_float4(v[4], v[5], v[6], v[7]);
}
__device__ __forceinline__ void st8(__nv_bfloat16* p, const float* v) {
  *(uint4*)p = make_uint4(pack2(v[0], v[1]), pack2(v[2], v[3]), pack2(v[4], v[5]), pack2(v[6], v[7]));
}
// X[t][d] = bf16(U[-1,1)) from (TAG_BERT_X, seed, EST) at counter (step*Te + tl)*D + d (bf16-exact, so the
// fp32 residual copy and the GEMM operand agree); target 0.5*U[-1,1)
__global__ void __launch_bounds__(256) data_kernel(uint64_t seed, int64_t step_h, const int64_t* step_dev, int est_base,
                                                   int Te, int D, int rows, float* X32, __nv_bfloat16* Xb,
                                                   float* target) {
  const int64_t step = cur_step(step_h, step_dev);
  const int t = blockIdx.x * 8 + (threadIdx.x >> 5), lane = threadIdx.x & 31;
  if (t >= rows) return;
  const int e = t / Te, tl = t - e * Te;
  const uint64_t sx = derive3(TAG_BERT_X, seed, (uint64_t)(est_base + e));
  const uint64_t sy = derive3(TAG_BERT_Y, seed, (uint64_t)(est_base + e));
  const uint64_t row0 = ((uint64_t)step * Te + tl) * (uint64_t)D;
  for (int col = lane * 8; col < D; col += 256) {
    float x[8], y[8];
#pragma unroll
    for (int q = 0; q < 8; ++q) {
      x[q] = __bfloat162float(__float2bfloat16_rn((float)(unit_float(draw_raw(sx, row0 + col + q)) * 2.0 - 1.0)));
      y[q] = 0.5f * (float)(unit_float(draw_raw(sy, row0 + col + q)) * 2.0 - 1.0);
    }
    st8(X32 + (size_t)t * D + col, x);
    st8(Xb + (size_t)t * D + col, x);
    st8(target + (size_t)t * D + col, y);
  }
}

// loss[e] = sum 0.5*(y - target)^2 / Te over the EST's rows (64 fixed element ranges, fixed
// tree, ranges summed in order); dy = bf16((y - target) / Te)
constexpr int MSE_THREADS = 256, MSE_BLOCKS = 64;
__global__ void __launch_bounds__(MSE_THREADS) mse_kernel(const float* __restrict__ y, const float* __restrict__ tgt,
                                                          int Te, int D, __nv_bfloat16* __restrict__ dy,
                                                          float* __restrict__ part) {
  const int e = blockIdx.y, blk = blockIdx.x;
  const int64_t per_est = (int64_t)Te * D;
  const int64_t chunk = (per_est + MSE_BLOCKS - 1) / MSE_BLOCKS;
  const int64_t lo = blk * chunk, hi = min(per_est, lo + chunk);
  const float inv = 1.f / (float)Te;
  float acc = 0.f;
  for (int64_t k = lo + threadIdx.x; k < hi; k += MSE_THREADS) {
    const int64_t i = (int64_t)e * per_est + k;
    const float diff = y[i] - tgt[i];
    dy[i] = __float2bfloat16_rn(diff * inv);
    acc += 0.5f * diff * diff;
  }
  __shared__ float sm[MSE_THREADS];
  sm[threadIdx.x] = acc;
  __syncthreads();
  for (int w = MSE_THREADS / 2; w > 0; w >>= 1) {
    if (threadIdx.x < w) sm[threadIdx.x] += sm[threadIdx.x + w];
    __syncthreads();
  }
  if (threadIdx.x == 0) part[e * MSE_BLOCKS + blk] = sm[0];
}
__global__ void mse_final_kernel(const float* __restrict__ part, int E, int Te, float* __restrict__ loss) {
  const int e = blockIdx.x * blockDim.x + threadIdx.x;
  if (e >= E) return;
  float acc = 0.f;
  for (int b = 0; b < MSE_BLOCKS; ++b) acc += part[e * MSE_BLOCKS + b];
  loss[e] = acc / (float)Te;
}

// bf16 operand copies of fp32 master weights: W [R][C] -> Wb [R][C] and Wt [C][R]
struct CastT {
  const float* w;
  __nv_bfloat16* wb;
  __nv_bfloat16* wt;
  int R, C;
};
constexpr int MAX_CAST = 64;
struct CastTable {
  CastT m[MAX_CAST];
  int n;
};
__global__ void __launch_bounds__(256) cast_t_kernel(const __grid_constant__ CastTable tab) {
  __shared__ float tile[64][65];
  const CastT& m = tab.m[blockIdx.z];
  const int r0 = blockIdx.y * 64, c0 = blockIdx.x * 64;
  if (r0 >= m.R || c0 >= m.C) return;
  const int tx = threadIdx.x & 31, ty = threadIdx.x >> 5;
  for (int k = ty; k < 64; k += 8) {
    const int r = r0 + k, c = c0 + 2 * tx;
    if (r < m.R && c + 1 < m.C) {
      const float2 v = *(const float2*)(m.w + (size_t)r * m.C + c);
      tile[k][2 * tx] = v.x;
      tile[k][2 * tx + 1] = v.y;
      *(uint32_t*)(m.wb + (size_t)r * m.C + c) = pack2(v.x, v.y);
    }
  }
  __syncthreads();
  for (int k = ty; k < 64; k += 8) {
    const int c = c0 + k, r = r0 + 2 * tx;
    if (c < m.C && r + 1 < m.R) *(uint32_t*)(m.wt + (size_t)c * m.R + r) = pack2(tile[2 * tx][k], tile[2 * tx + 1][k]);
  }
}

}  // namespace bert

// ----------------------------------------------------------------- launchers
int attn_fwd_tc_launch(const void* qkv, void* out, int n_seq, int Dm, int H, int seqs_per_est, int est_base, int L,
                       int layer, uint64_t seed, int64_t step, float p, const int64_t* step_dev, cudaStream_t s,
                       float* stats, uint32_t* mbits);
int attn_bwd_tc_launch(const void* qkv, const void* dctx, void* dqkv, int n_seq, int Dm, int H, int seqs_per_est,
                       int est_base, int L, int layer, uint64_t seed, int64_t step, float p, const int64_t* step_dev,
                       cudaStream_t s, const float* stats, const uint32_t* mbits);
static bool attn_tc_enabled() {  // BT_ATTN_TC=0: the mma.sync forward (bt_bert.cu) instead of bt_attn_tc.cu
  const char* e = getenv("BT_ATTN_TC");
  return !(e && e[0] == '0');
}
static int ok_or_cuda_b() { return cudaGetLastError() == cudaSuccess ? OK : ERR_CUDA; }

int bert_attn_launch(int backward, const void* qkv, const void* dctx, void* out, int n_seq, int Dm, int H,
                     int seqs_per_est, int est_base, int L, int layer, uint64_t seed, int64_t step, float p,
                     const int64_t* step_dev, cudaStream_t s, float* stats, uint32_t* mbits) {
  bert::AttnArgs a{(const __nv_bfloat16*)qkv, (const __nv_bfloat16*)dctx, (__nv_bfloat16*)out, Dm, H, seqs_per_est,
                   est_base, L, layer, n_seq * H, seed, step, p, step_dev};
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  if (attn_tc_enabled())
    return backward ? attn_bwd_tc_launch(qkv, dctx, out, n_seq, Dm, H, seqs_per_est, est_base, L, layer, seed, step, p,
                                         step_dev, s, stats, mbits)
                    : attn_fwd_tc_launch(qkv, out, n_seq, Dm, H, seqs_per_est, est_base, L, layer, seed, step, p,
                                         step_dev, s, stats, mbits);
  if (!backward) {
    static bool attr = false;
    if (!attr) {
      if (cudaFuncSetAttribute(bert::attn_fwd_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, bert::ATF_SMEM) !=
              cudaSuccess ||
          cudaFuncSetAttribute(bert::attn_fwd_kernel, cudaFuncAttributePreferredSharedMemoryCarveout, 100) !=
              cudaSuccess)
        return ERR_CUDA;
      attr = true;
    }
    const int grid = a.n_items < 2 * sms ? a.n_items : 2 * sms;
    bert::attn_fwd_kernel<<<grid, bert::AT_THREADS, bert::ATF_SMEM, s>>>(a);
  } else {
    static bool attr = false;
    if (!attr) {
      if (cudaFuncSetAttribute(bert::attn_bwd_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, bert::ATB_SMEM) !=
              cudaSuccess ||
          cudaFuncSetAttribute(bert::attn_bwd_kernel, cudaFuncAttributePreferredSharedMemoryCarveout, 100) !=
              cudaSuccess)
        return ERR_CUDA;
      attr = true;
    }
    const int grid = a.n_items < sms ? a.n_items : sms;
    bert::attn_bwd_kernel<<<grid, bert::AT_THREADS, bert::ATB_SMEM, s>>>(a);
  }
  return ok_or_cuda_b();
}

template <class K>
static bool smem_attr(K kern, int bytes) {
  return cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes) == cudaSuccess;
}
template <int NC>
static int ln_launch_nc(int backward, const bert::LnArgs& a, cudaStream_t s) {
  static int sms = 0;
  if (!sms) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  }
  if (!backward) {
    constexpr int smem = bert::LnfSlot<NC>::PAR + 2 * bert::LNF_WARPS * bert::LnfSlot<NC>::BYTES;
    static bool attr = false;
    if (!attr && !(attr = smem_attr(bert::ln_fwd_kernel<NC>, smem))) return ERR_CUDA;
    const int warps = (a.rows + 7) / 8;  // ~8 rows per warp at most, as many blocks as fit resident
    const int per_sm = (227 * 1024) / (smem + 1024);
    int grid = (warps + bert::LNF_WARPS - 1) / bert::LNF_WARPS;
    if (grid > per_sm * sms) grid = per_sm * sms;
    bert::ln_fwd_kernel<NC><<<grid, 32 * bert::LNF_WARPS, smem, s>>>(a);
  } else if (a.resid) {
    constexpr int smem = 256 * NC * 4 + 2 * bert::LNB_WARPS * bert::LnbSlot<NC, true>::BYTES;
    static bool attr = false;
    if (!attr && !(attr = smem_attr(bert::ln_bwd_kernel<NC, true>, smem))) return ERR_CUDA;
    bert::ln_bwd_kernel<NC, true><<<a.rows / bert::LN_CHUNK, 32 * bert::LNB_WARPS, smem, s>>>(a);
  } else {
    constexpr int smem = 256 * NC * 4 + 2 * bert::LNB_WARPS * bert::LnbSlot<NC, false>::BYTES;
    static bool attr = false;
    if (!attr && !(attr = smem_attr(bert::ln_bwd_kernel<NC, false>, smem))) return ERR_CUDA;
    bert::ln_bwd_kernel<NC, false><<<a.rows / bert::LN_CHUNK, 32 * bert::LNB_WARPS, smem, s>>>(a);
  }
  return ok_or_cuda_b();
}

// forward: resid (fp32) / branch (bf16) / bias / gamma / beta -> xsum, stats, y32, yb
// backward: dy2 (in1, fp32, may be null), dy1 (in2, bf16), xsum, stats_in, gamma -> dx (y32), dbranch (yb), part
int bert_ln_launch(int backward, const float* in1, const void* in2, const float* bias, const float* gamma,
                   const float* beta, float* xsum, float* stats, float* y32, void* yb, float* part, int E, int Te,
                   int D, int est_base, int L, int layer, int site, uint64_t seed, int64_t step, float p, float eps,
                   const int64_t* step_dev, cudaStream_t s, const float* rx, const float* rst, const float* rg,
                   const float* rb) {
  if (D % 256 || D > 1024 || Te % bert::LN_CHUNK) return ERR_INPUT;
  bert::LnArgs a{};
  a.resid = in1;
  a.rx = rx;
  a.rst = (const float2*)rst;
  a.rg = rg;
  a.rb = rb;
  a.bin = (const __nv_bfloat16*)in2;
  a.bias = bias;
  a.gamma = gamma;
  a.beta = beta;
  a.xsum = xsum;
  a.stats_in = (const float2*)stats;
  a.stats = (float2*)stats;
  a.y32 = y32;
  a.yb = (__nv_bfloat16*)yb;
  a.part = part;
  a.D = D;
  a.Te = Te;
  a.rows = E * Te;
  a.est_base = est_base;
  a.L = L;
  a.layer = layer;
  a.site = site;
  a.seed = seed;
  a.step = step;
  a.step_dev = step_dev;
  a.p = p;
  a.eps = eps;
  switch (D / 256) {
    case 1: return ln_launch_nc<1>(backward, a, s);
    case 2: return ln_launch_nc<2>(backward, a, s);
    case 3: return ln_launch_nc<3>(backward, a, s);
    default: return ln_launch_nc<4>(backward, a, s);
  }
}

int bert_ln_fold_launch(const float* part, int E, int Te, int D, float* dg, float* db, float* dr, int64_t est_stride,
                        cudaStream_t s) {
  if (Te % bert::LN_CHUNK) return ERR_INPUT;
  if (est_stride % 4 || ((uintptr_t)dg | (uintptr_t)db | (uintptr_t)dr) & 15) return ERR_INPUT;  // 16-byte stores
  bert::ln_fold_kernel<<<dim3((3 * D + 127) / 128, E), 32 * bert::LNF_SEGS, 0, s>>>(part, Te / bert::LN_CHUNK, D, dg,
                                                                                   db, dr, est_stride);
  return ok_or_cuda_b();
}

int bert_data_launch(uint64_t seed, int64_t step, int est_base, int E, int Te, int D, float* X32, void* Xb,
                     float* target, const int64_t* step_dev, cudaStream_t s) {
  if (D % 8) return ERR_INPUT;
  const int rows = E * Te;
  bert::data_kernel<<<(rows + 7) / 8, 256, 0, s>>>(seed, step, step_dev, est_base, Te, D, rows, X32,
                                                   (__nv_bfloat16*)Xb, target);
  return ok_or_cuda_b();
}

int bert_mse_launch(const float* y, const float* tgt, int E, int Te, int D, void* dy, float* part, float* loss,
                    cudaStream_t s) {
  bert::mse_kernel<<<dim3(bert::MSE_BLOCKS, E), bert::MSE_THREADS, 0, s>>>(y, tgt, Te, D, (__nv_bfloat16*)dy, part);
  bert::mse_final_kernel<<<(E + 127) / 128, 128, 0, s>>>(part, E, Te, loss);
  return ok_or_cuda_b();
}

int bert_cast_weights_launch(const float* const* w, void* const* wb, void* const* wt, const int* R, const int* C, int n,
                             cudaStream_t s) {
  if (n < 1 || n > bert::MAX_CAST) return ERR_INPUT;
  bert::CastTable tab{};
  int maxr = 0, maxc = 0;
  for (int i = 0; i < n; ++i) {
    if (R[i] % 2 || C[i] % 2) return ERR_INPUT;
    tab.m[i] = bert::CastT{w[i], (__nv_bfloat16*)wb[i], (__nv_bfloat16*)wt[i], R[i], C[i]};
    maxr = R[i] > maxr ? R[i] : maxr;
    maxc = C[i] > maxc ? C[i] : maxc;
  }
  tab.n = n;
  bert::cast_t_kernel<<<dim3((maxc + 63) / 64, (maxr + 63) / 64, n), 256, 0, s>>>(tab);
  return ok_or_cuda_b();
}

}  // namespace bt
