// bt_attn_tc.cu -- BERT attention forward on the 5th-generation tensor cores (C4).
//
// One (sequence, head) item per iteration of a persistent CTA of 4 warps; thread i owns query row i:
//   TMA      Q, K [128][64] (K-major, 128 B swizzle) and V as two MN-major 64x64 boxes;
//   tcgen05  S = Q K^T (M = 128, N = 128, K = 64) into TMEM columns [0, 128);
//   softmax  each thread loads ITS row of S from TMEM (tcgen05.ld: max, exp2 row sum in column order,
//            then P -- three passes, few registers), applies the attention-probability dropout keyed
//            exactly as the mma.sync kernel keys it (bt_bert.cu: one splitmix64 draw per (16-row
//            block, row, column pair), 16-bit fields; rows i and i^8 share a draw, computed by one
//            of the two lanes and exchanged by shuffle), and writes the bf16 row of P into a K-major
//            swizzled shared tile;
//   tcgen05  O = P V (M = 128, N = 64, K = 128; V MN-major) into TMEM columns [0, 64) (S's, consumed);
//   store    each thread its row of O (bf16).
// Every output element is produced by a fixed instruction sequence over its own inputs: the bits do
// not depend on the grid, the item order or which ESTs share the launch.
#include <cuda.h>
#include <cuda_bf16.h>
#include <cuda_runtime.h>
#include <stdint.h>

#include "bt_common.cuh"
#include "bt_tc.cuh"

namespace bt {
bool make_map(CUtensorMap* map, const void* ptr, int rows, int K, int box_rows, int batch, int64_t bstride);
bool make_map_mn(CUtensorMap* map, const void* ptr, int rows, int K, int batch, int64_t bstride);

namespace attn_tc {
using namespace tc;

constexpr uint64_t TAG_BERT_ADROP = 0x4245'5254'4144'5250ull;  // == bt_bert.cu (same masks)
constexpr int SEQ = 128, HD = 64, THREADS = 128;
// P (bf16, two K-major k-blocks) reuses the Q/K tiles once the S product has consumed them; O reuses
// S's TMEM columns once every thread holds its row statistics: 48 KB + 128 TMEM columns per CTA, so
// four CTAs (16 warps) share an SM and hide each other's load / MMA / softmax latency.
constexpr int OFF_Q = 0, OFF_K = 16384, OFF_P = 0, OFF_V = 32768, OFF_BAR = 49152;
constexpr int SMEM = OFF_BAR + 64 + 1024;  // + alignment slack
constexpr int TMEM_COLS = 128;             // S: [0, 128); then O: [0, 64)

struct Args {
  __nv_bfloat16* out;  // ctx [T][Dm]
  int Dm, H, seqs_per_est, est_base, L, layer, n_items;
  uint64_t seed;
  int64_t step;
  float p;
  const int64_t* step_dev;
  float2* stats;  // [n_items][128] (nm, inv) of every query row for the backward, or NULL
  uint32_t* mbits;  // [n_items][128][4] keep bits of every row (column c at word c / 32, bit c % 32), or NULL
};

__device__ __forceinline__ float ex2_approx(float x) {
  float y;
  asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}
typedef unsigned long long f32x2;  // packed fp32 pair (sm_100a FADD2 / FMUL2 / FFMA2)
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
__device__ __forceinline__ uint32_t pack2(float lo, float hi) {
  const __nv_bfloat162 v = __floats2bfloat162_rn(lo, hi);
  return *(const uint32_t*)&v;
}

// This thread's softmax row statistics from S in TMEM columns [0, 128) of its lane: nm = -max(x*SC)
// and inv = 1 / sum exp2(x*SC + nm), the sum in column order (exp2 arguments as one FMA; MUFU ex2
// directly: arguments are <= 0).  The forward and the backward call this same sequence: same bits.
constexpr float SC = 0.125f * 1.4426950408889634f;  // 1/sqrt(64) * log2(e)
// (The 32-column slice loops are not unrolled: the attention kernels are large and their four CTAs per SM
// run different phases -- the instruction cache, not the ALU, was the forward's limit.)
__device__ __forceinline__ void row_stats(uint32_t lane_base, float* nm_out, float* inv_out) {
  float mx = -INFINITY;
#pragma unroll 1
  for (int c = 0; c < SEQ / 32; ++c) {
    uint32_t v[32];
    tmem_ld32(lane_base + c * 32, v);
    tmem_ld_wait();
#pragma unroll
    for (int q = 0; q < 32; ++q) mx = fmaxf(mx, __uint_as_float(v[q]));
  }
  const float nm = -__fmul_rn(mx, SC);
  float l[2] = {0.f, 0.f};  // the two 64-column halves, each in column order, then added
#pragma unroll
  for (int h = 0; h < 2; ++h) {
#pragma unroll 1
    for (int c = 2 * h; c < 2 * h + 2; ++c) {
      uint32_t v[32];
      tmem_ld32(lane_base + c * 32, v);
      tmem_ld_wait();
#pragma unroll
      for (int q = 0; q < 32; ++q) l[h] += ex2_approx(__fmaf_rn(__uint_as_float(v[q]), SC, nm));
    }
  }
  *nm_out = nm;
  *inv_out = 1.f / (l[0] + l[1]);
}
// The same statistics from one 64-column half (cols [64*hf, 64*hf + 64)) per thread, the halves of a
// row combined through shared memory: identical bits to row_stats (max is exact; sum = half0 + half1).
__device__ __forceinline__ void row_stats_half(uint32_t lane_base, int hf, int row, float* red, float* nm_out,
                                               float* inv_out) {
  float mx = -INFINITY;
#pragma unroll
  for (int c = 0; c < 2; ++c) {
    uint32_t v[32];
    tmem_ld32(lane_base + hf * 64 + c * 32, v);
    tmem_ld_wait();
#pragma unroll
    for (int q = 0; q < 32; ++q) mx = fmaxf(mx, __uint_as_float(v[q]));
  }
  red[hf * SEQ + row] = mx;
  __syncthreads();
  mx = fmaxf(red[row], red[SEQ + row]);
  const float nm = -__fmul_rn(mx, SC);
  float l = 0.f;
#pragma unroll
  for (int c = 0; c < 2; ++c) {
    uint32_t v[32];
    tmem_ld32(lane_base + hf * 64 + c * 32, v);
    tmem_ld_wait();
#pragma unroll
    for (int q = 0; q < 32; ++q) l += ex2_approx(__fmaf_rn(__uint_as_float(v[q]), SC, nm));
  }
  __syncthreads();  // everyone has read the max slots
  red[hf * SEQ + row] = l;
  __syncthreads();
  *nm_out = nm;
  *inv_out = 1.f / (red[row] + red[SEQ + row]);
}
// The 16 mask fields (one per column pair) of this row's 32-column slice c: rows i and i^8 share a
// draw; each of the two lanes computes half of the slice's draws and they exchange by shuffle.
__device__ __forceinline__ void row_fields(uint64_t sd, uint64_t nb, int c, int hi, uint32_t thr, uint32_t* f) {
  const int fsh = hi * 32;
#pragma unroll
  for (int t = 0; t < 8; ++t) {
    uint64_t r = 0;
    if (thr) r = draw_raw(sd, nb + (uint64_t)(c * 16 + 2 * t + hi));
    const uint64_t o = __shfl_xor_sync(0xffffffffu, r, 8);  // the partner row's draw: pair 2t + !hi
    const uint64_t r_even = hi ? o : r, r_odd = hi ? r : o;
    f[2 * t] = (uint32_t)(r_even >> fsh);
    f[2 * t + 1] = (uint32_t)(r_odd >> fsh);
  }
}

__global__ void __launch_bounds__(THREADS, 4)
    attn_fwd_tc_kernel(const __grid_constant__ CUtensorMap mqk, const __grid_constant__ CUtensorMap mv, const Args a) {
  extern __shared__ uint8_t smem_raw[];
  const uint32_t raw = su32(smem_raw), base = (raw + 1023u) & ~1023u;
  uint8_t* const gbase = smem_raw + (base - raw);
  const uint32_t bar_ld = base + OFF_BAR, bar_s = bar_ld + 8, bar_o = bar_ld + 16;
  uint32_t* const tmem_slot = (uint32_t*)(gbase + OFF_BAR + 32);
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  if (tid == 0) {
    asm volatile("prefetch.tensormap [%0];" ::"l"(&mqk) : "memory");
    asm volatile("prefetch.tensormap [%0];" ::"l"(&mv) : "memory");
    mbar_init(bar_ld, 1);
    mbar_init(bar_s, 1);
    mbar_init(bar_o, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(su32(tmem_slot)),
                 "r"(TMEM_COLS)
                 : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;
  const uint32_t lane_base = tmem + ((uint32_t)(warp * 32) << 16);  // this warp's TMEM lane quarter
  const int64_t step = a.step_dev ? *a.step_dev : a.step;
  const uint32_t thr = a.p > 0.f ? (uint32_t)ceil((double)a.p * 65536.0) : 0u;
  const float keep = a.p < 1.f ? 1.f / (1.f - a.p) : 0.f;
  const int hi = (tid >> 3) & 1;                       // rows i, i^8 share draws (lanes l, l^8)
  auto load_item = [&](int it) {  // Q, K, V of item `it` (thread 0)
    const int s = it / a.H, h = it - (it / a.H) * a.H;
    mbar_arrive_expect_tx(bar_ld, 3 * 16384);
    tma_load_3d(base + OFF_Q, &mqk, h * HD, s * SEQ, 0, bar_ld);
    tma_load_3d(base + OFF_K, &mqk, a.Dm + h * HD, s * SEQ, 0, bar_ld);
    tma_load_3d(base + OFF_V, &mv, 2 * a.Dm + h * HD, s * SEQ, 0, bar_ld);
    tma_load_3d(base + OFF_V + 8192, &mv, 2 * a.Dm + h * HD, s * SEQ + 64, 0, bar_ld);
  };
  if (tid == 0 && (int)blockIdx.x < a.n_items) load_item(blockIdx.x);
  int n = 0;
  for (int it = blockIdx.x; it < a.n_items; it += gridDim.x, ++n) {
    const int s = it / a.H, h = it - (it / a.H) * a.H;
    const uint32_t ph = n & 1;
    if (tid == 0) {
      mbar_wait(bar_ld, ph);
      tc_fence_after();
      constexpr uint32_t idS = idesc_bf16(128, 128, false, false);
      const uint64_t dq = kmajor_sw128_desc(base + OFF_Q), dk = kmajor_sw128_desc(base + OFF_K);
#pragma unroll
      for (int k = 0; k < HD / 16; ++k) tc_mma(tmem, dq + 2 * k, dk + 2 * k, idS, k != 0);
      tc_commit(bar_s);
    }
    mbar_wait(bar_s, ph);
    tc_fence_after();
    // this thread's row of S, three passes over TMEM (row max; exp2 row sum in column order; P)
    float nm, inv;
    row_stats(lane_base, &nm, &inv);
    if (a.stats) a.stats[(size_t)it * SEQ + tid] = make_float2(nm, inv);  // the backward reuses them (same bits)
    // dropout keyed by (EST, step, layer, sequence, head, row, column pair) -- bt_bert.cu's layout
    const int e = s / a.seqs_per_est, sl = s - e * a.seqs_per_est;
    const uint64_t sd = derive3(TAG_BERT_ADROP, a.seed, (uint64_t)(a.est_base + e));
    const uint64_t nb = ((((uint64_t)step * a.L + a.layer) * a.seqs_per_est + sl) * a.H + h) * (uint64_t)(SEQ * SEQ / 4) +
                        (uint64_t)((tid >> 4) * 8 + (tid & 7)) * 64;
    uint8_t* const prow = gbase + OFF_P + tid * 128;
    uint32_t* const kbits = a.mbits ? a.mbits + ((size_t)it * SEQ + tid) * 4 : nullptr;
#pragma unroll 1
    for (int c = 0; c < SEQ / 32; ++c) {  // 32 columns = 16 column pairs; this lane draws 8, its partner 8
      uint32_t v[32];
      tmem_ld32(lane_base + c * 32, v);
      tmem_ld_wait();
      uint32_t f[16];
      row_fields(sd, nb, c, hi, thr, f);
      const int kb = c >> 1;
      uint32_t bits = 0;
#pragma unroll
      for (int cc = 0; cc < 4; ++cc) {  // four 16-byte chunks (8 columns each) of this 32-column slice
        uint32_t w[4];
#pragma unroll
        for (int hh = 0; hh < 4; ++hh) {
          const int q = cc * 8 + 2 * hh;  // column c*32 + q, pair index q / 2
          const float p0 = ex2_approx(__fmaf_rn(__uint_as_float(v[q]), SC, nm)) * inv;
          const float p1 = ex2_approx(__fmaf_rn(__uint_as_float(v[q + 1]), SC, nm)) * inv;
          float m0 = 1.f, m1 = 1.f;
          if (thr) {
            const bool k0 = !((f[q >> 1] & 0xFFFFu) < thr), k1 = !((f[q >> 1] >> 16) < thr);
            m0 = k0 ? keep : 0.f;
            m1 = k1 ? keep : 0.f;
            bits |= (k0 ? 1u : 0u) << q;
            bits |= (k1 ? 1u : 0u) << (q + 1);
          }
          w[hh] = pack2(p0 * m0, p1 * m1);
        }
        const int chunk = (c & 1) * 4 + cc;  // 16-byte chunk within the 128-byte row of k-block kb
        *(uint4*)(prow + kb * 16384 + ((chunk ^ (tid & 7)) << 4)) = make_uint4(w[0], w[1], w[2], w[3]);
      }
      if (kbits) kbits[c] = bits;  // the keep bits for the backward (which then draws nothing)
    }
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");  // P visible to the tensor core
    tc_fence_before();
    __syncthreads();
    if (tid == 0) {
      tc_fence_after();
      constexpr uint32_t idO = idesc_bf16(128, HD, false, true);
      const uint64_t dv = mnmajor_sw128_desc(base + OFF_V);
#pragma unroll
      for (int kb = 0; kb < 2; ++kb) {
        const uint64_t dp = kmajor_sw128_desc(base + OFF_P + kb * 16384);
#pragma unroll
        for (int k = 0; k < 4; ++k)
          tc_mma(tmem, dp + 2 * k, dv + (uint64_t)(kb * 4 + k) * (2048 >> 4), idO, (kb | k) != 0);
      }
      tc_commit(bar_o);
    }
    mbar_wait(bar_o, ph);
    tc_fence_after();
    // the O product has consumed P and V: the shared tiles are free, so the next item's loads overlap
    // this item's output drain
    if (tid == 0 && it + (int)gridDim.x < a.n_items) load_item(it + gridDim.x);
    uint4* const orow = (uint4*)(a.out + ((size_t)s * SEQ + tid) * a.Dm + h * HD);
#pragma unroll
    for (int c = 0; c < HD / 32; ++c) {
      uint32_t v[32];
      tmem_ld32(lane_base + c * 32, v);
      tmem_ld_wait();
#pragma unroll
      for (int q = 0; q < 4; ++q)
        orow[c * 4 + q] =
            make_uint4(pack2(__uint_as_float(v[8 * q]), __uint_as_float(v[8 * q + 1])),
                       pack2(__uint_as_float(v[8 * q + 2]), __uint_as_float(v[8 * q + 3])),
                       pack2(__uint_as_float(v[8 * q + 4]), __uint_as_float(v[8 * q + 5])),
                       pack2(__uint_as_float(v[8 * q + 6]), __uint_as_float(v[8 * q + 7])));
    }
    tc_fence_before();
    __syncthreads();  // TMEM and the shared tiles are free for the next item
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 0) {
    tc_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(TMEM_COLS) : "memory");
  }
}


// ---------------------------------------------------------------------------------------- backward
// Per (sequence, head) item; 8 warps, thread (row i, half hf) owns columns [64 hf, 64 hf + 64) of query
// row i for the row work and of key row i for dK / dV (row reductions combined through shared memory):
//   TMA      Q, K, V, dO [128][64] K-major tiles (each tile is also read MN-major by the products
//            that need its transpose: the bytes of a K-major [r][64] tile are the MN-major layout of
//            its [64][r] view);
//   tcgen05  S = Q K^T -> TMEM [0,128), dPd = dO V^T -> TMEM [128,256);
//   rows     P recomputed by the forward's exact sequence (row_stats), masks, dP = dPd * mask,
//            D = sum dP*P (column order), dS = P (dP - D) / 8 -> shared (K-major [q][key]);
//            the dropped P kept packed in registers;
//   tcgen05  dQ = dS K -> [0,64), dK = dS^T Q -> [64,128); then Pd (from registers) replaces dS in
//            shared memory and dV = Pd^T dO -> [128,192);
//   store    dq / dk / dv rows into dqkv (bf16).
constexpr int B_OFF_Q = 0, B_OFF_K = 16384, B_OFF_V = 32768, B_OFF_DO = 49152, B_OFF_S = 65536, B_OFF_RED = 98304,
              B_OFF_BAR = B_OFF_RED + 2 * SEQ * 4;
constexpr int B_SMEM = B_OFF_BAR + 64 + 1024;
constexpr int B_TMEM_COLS = 256;
constexpr int B_THREADS = 256;  // thread (row, half): row = 32 * (warp % 4) + lane, columns [64*half, +64)

// MN-major SW128 descriptor with an explicit distance between 64-wide MN blocks
__device__ __forceinline__ uint64_t mn_desc(uint32_t saddr, uint32_t lbo) {
  return (uint64_t)((saddr & 0x3FFFF) >> 4) | ((uint64_t)(lbo >> 4) << 16) | ((uint64_t)(1024 >> 4) << 32) |
         ((uint64_t)1 << 46) | ((uint64_t)2 << 61);
}

struct BwdArgs {
  __nv_bfloat16* dqkv;  // [T][3*Dm]
  int Dm, H, seqs_per_est, est_base, L, layer, n_items;
  uint64_t seed;
  int64_t step;
  float p;
  const int64_t* step_dev;
  const float2* stats;  // the forward's row statistics [n_items][128], or NULL: recompute them
  const uint32_t* mbits;  // the forward's keep bits [n_items][128][4], or NULL: draw the masks again
};

// 32 TMEM columns of this lane's row -> 32 bf16 (64 bytes) at dst
__device__ __forceinline__ void store_row32(__nv_bfloat16* dst, uint32_t taddr) {
  uint4* const o = (uint4*)dst;
  uint32_t v[32];
  tmem_ld32(taddr, v);
  tmem_ld_wait();
#pragma unroll
  for (int q = 0; q < 4; ++q)
    o[q] = make_uint4(pack2(__uint_as_float(v[8 * q]), __uint_as_float(v[8 * q + 1])),
                      pack2(__uint_as_float(v[8 * q + 2]), __uint_as_float(v[8 * q + 3])),
                      pack2(__uint_as_float(v[8 * q + 4]), __uint_as_float(v[8 * q + 5])),
                      pack2(__uint_as_float(v[8 * q + 6]), __uint_as_float(v[8 * q + 7])));
}

__global__ void __launch_bounds__(B_THREADS, 2)
    attn_bwd_tc_kernel(const __grid_constant__ CUtensorMap mqk, const __grid_constant__ CUtensorMap mdo,
                       const BwdArgs a) {
  extern __shared__ uint8_t smem_raw[];
  const uint32_t raw = su32(smem_raw), base = (raw + 1023u) & ~1023u;
  uint8_t* const gbase = smem_raw + (base - raw);
  float* const red = (float*)(gbase + B_OFF_RED);  // [2 halves][128 rows] row-reduction exchange
  const uint32_t bar_ld = base + B_OFF_BAR, bar_s = bar_ld + 8, bar_a = bar_ld + 16, bar_v = bar_ld + 24;
  uint32_t* const tmem_slot = (uint32_t*)(gbase + B_OFF_BAR + 40);
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int hf = warp >> 2, row = (warp & 3) * 32 + lane;
  if (tid == 0) {
    asm volatile("prefetch.tensormap [%0];" ::"l"(&mqk) : "memory");
    asm volatile("prefetch.tensormap [%0];" ::"l"(&mdo) : "memory");
    mbar_init(bar_ld, 1);
    mbar_init(bar_s, 1);
    mbar_init(bar_a, 1);
    mbar_init(bar_v, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(su32(tmem_slot)),
                 "r"(B_TMEM_COLS)
                 : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;
  const uint32_t lane_base = tmem + ((uint32_t)((warp & 3) * 32) << 16);  // this warp's TMEM lane quarter
  const int64_t step = a.step_dev ? *a.step_dev : a.step;
  const uint32_t thr = a.p > 0.f ? (uint32_t)ceil((double)a.p * 65536.0) : 0u;
  const float keep = a.p < 1.f ? 1.f / (1.f - a.p) : 0.f;
  const int hi = (row >> 3) & 1;  // rows i, i^8 (lanes l, l^8 of one warp) share draws
  const int ld = 3 * a.Dm;
  // the next item's Q, K, V load as soon as the dQ / dK products have consumed this item's (bar_a), its
  // dO once dV has (bar_v): one expect_tx of all four tiles per item (thread 0)
  auto load_qkv = [&](int it) {
    const int s = it / a.H, h = it - (it / a.H) * a.H;
    mbar_arrive_expect_tx(bar_ld, 4 * 16384);
    tma_load_3d(base + B_OFF_Q, &mqk, h * HD, s * SEQ, 0, bar_ld);
    tma_load_3d(base + B_OFF_K, &mqk, a.Dm + h * HD, s * SEQ, 0, bar_ld);
    tma_load_3d(base + B_OFF_V, &mqk, 2 * a.Dm + h * HD, s * SEQ, 0, bar_ld);
  };
  auto load_do = [&](int it) {
    const int s = it / a.H, h = it - (it / a.H) * a.H;
    tma_load_3d(base + B_OFF_DO, &mdo, h * HD, s * SEQ, 0, bar_ld);
  };
  if (tid == 0 && (int)blockIdx.x < a.n_items) {
    load_qkv(blockIdx.x);
    load_do(blockIdx.x);
  }
  int n = 0;
  for (int it = blockIdx.x; it < a.n_items; it += gridDim.x, ++n) {
    const int s = it / a.H, h = it - (it / a.H) * a.H;
    const uint32_t ph = n & 1;
    const bool more = it + (int)gridDim.x < a.n_items;
    if (tid == 0) {
      mbar_wait(bar_ld, ph);
      tc_fence_after();
      constexpr uint32_t id128 = idesc_bf16(128, 128, false, false);
      const uint64_t dq = kmajor_sw128_desc(base + B_OFF_Q), dk = kmajor_sw128_desc(base + B_OFF_K);
      const uint64_t dv = kmajor_sw128_desc(base + B_OFF_V), ddo = kmajor_sw128_desc(base + B_OFF_DO);
#pragma unroll
      for (int k = 0; k < HD / 16; ++k) tc_mma(tmem, dq + 2 * k, dk + 2 * k, id128, k != 0);         // S
#pragma unroll
      for (int k = 0; k < HD / 16; ++k) tc_mma(tmem + 128, ddo + 2 * k, dv + 2 * k, id128, k != 0);  // dPd
      tc_commit(bar_s);
    }
    // the forward's statistics and keep bits of this row, in flight while the products run
    float2 st = make_float2(0.f, 0.f);
    uint2 mb = make_uint2(0u, 0u);
    if (a.stats) st = a.stats[(size_t)it * SEQ + row];
    if (a.mbits) mb = *(const uint2*)(a.mbits + ((size_t)it * SEQ + row) * 4 + hf * 2);
    mbar_wait(bar_s, ph);
    tc_fence_after();
    float nm, inv;
    if (a.stats) {  // the same instruction sequence on the same S gave them: the same bits
      nm = st.x;
      inv = st.y;
    } else {
      row_stats_half(lane_base, hf, row, red, &nm, &inv);
    }
    const int e = s / a.seqs_per_est, sl = s - e * a.seqs_per_est;
    const uint64_t sd = derive3(TAG_BERT_ADROP, a.seed, (uint64_t)(a.est_base + e));
    const uint64_t nb = ((((uint64_t)step * a.L + a.layer) * a.seqs_per_est + sl) * a.H + h) * (uint64_t)(SEQ * SEQ / 4) +
                        (uint64_t)((row >> 4) * 8 + (row & 7)) * 64;
    // pass 3 (this half): dropped P (packed, registers), the keep bits (the forward's, or drawn again),
    // partial D = sum dP * P; P and dP * mask go back into TMEM in place of S and dPd for pass 4
    uint32_t pd[32], mbits[2] = {mb.x, mb.y};
    f32x2 D2 = pk2(0.f, 0.f);
    const f32x2 SC2 = pk2(SC, SC);
#pragma unroll
    for (int c2 = 0; c2 < 2; ++c2) {
      const int c = hf * 2 + c2;  // 32-column slice
      uint32_t v[32], g[32];
      tmem_ld32(lane_base + c * 32, v);
      tmem_ld32(lane_base + 128 + c * 32, g);
      tmem_ld_wait();
      if (!a.mbits) {
        uint32_t f[16];
        row_fields(sd, nb, c, hi, thr, f);
        uint32_t bits = 0;
#pragma unroll
        for (int q = 0; q < 32; q += 2) {
          bits |= (!((f[q >> 1] & 0xFFFFu) < thr) ? 1u : 0u) << q;
          bits |= (!((f[q >> 1] >> 16) < thr) ? 1u : 0u) << (q + 1);
        }
        mbits[c2] = bits;
      }
      // packed fp32 pairs (FFMA2 / FMUL2: the same per-element operations as the forward's P); D accumulates
      // as an (even, odd) column pair of FMAs, added at the end
      const uint32_t mw = mbits[c2];
#pragma unroll
      for (int q = 0; q < 32; q += 2) {
        const float2 t = upk2(fma2(pk2(__uint_as_float(v[q]), __uint_as_float(v[q + 1])), SC2, pk2(nm, nm)));
        const f32x2 pp = mul2(pk2(ex2_approx(t.x), ex2_approx(t.y)), pk2(inv, inv));
        const float m0 = thr ? (((mw >> q) & 1u) ? keep : 0.f) : 1.f;
        const float m1 = thr ? (((mw >> (q + 1)) & 1u) ? keep : 0.f) : 1.f;
        const f32x2 mm = pk2(m0, m1);
        const float2 pm = upk2(mul2(pp, mm));
        pd[c2 * 16 + (q >> 1)] = pack2(pm.x, pm.y);
        const f32x2 gm = mul2(pk2(__uint_as_float(g[q]), __uint_as_float(g[q + 1])), mm);
        D2 = fma2(gm, pp, D2);
        const float2 pf = upk2(pp), gf = upk2(gm);
        v[q] = __float_as_uint(pf.x);
        v[q + 1] = __float_as_uint(pf.y);
        g[q] = __float_as_uint(gf.x);
        g[q + 1] = __float_as_uint(gf.y);
      }
      tmem_st32(lane_base + c * 32, v);
      tmem_st32(lane_base + 128 + c * 32, g);
    }
    tmem_st_wait();
    const float2 Dp = upk2(D2);
    float D = Dp.x + Dp.y;
    if (!a.stats) __syncthreads();  // the sum slots of row_stats_half are read
    red[hf * SEQ + row] = D;
    __syncthreads();
    D = red[row] + red[SEQ + row];  // (half 0 + half 1)
    // pass 4: dS = P (dP - D) / 8 -> shared, K-major [q][key]: this half is k-block hf
    uint8_t* const srow = gbase + B_OFF_S + hf * 16384 + row * 128;
#pragma unroll
    for (int c2 = 0; c2 < 2; ++c2) {
      const int c = hf * 2 + c2;
      uint32_t v[32], g[32];
      tmem_ld32(lane_base + c * 32, v);        // P
      tmem_ld32(lane_base + 128 + c * 32, g);  // dP * mask
      tmem_ld_wait();
      const f32x2 DD = pk2(D, D), E8 = pk2(0.125f, 0.125f);
#pragma unroll
      for (int cc = 0; cc < 4; ++cc) {
        uint32_t w[4];
#pragma unroll
        for (int hh = 0; hh < 4; ++hh) {  // (P (dP m - D)) / 8, packed pairs
          const int q = cc * 8 + 2 * hh;
          const f32x2 pp = pk2(__uint_as_float(v[q]), __uint_as_float(v[q + 1]));
          const float2 ds = upk2(mul2(mul2(pp, sub2(pk2(__uint_as_float(g[q]), __uint_as_float(g[q + 1])), DD)), E8));
          w[hh] = pack2(ds.x, ds.y);
        }
        const int chunk = c2 * 4 + cc;
        *(uint4*)(srow + ((chunk ^ (row & 7)) << 4)) = make_uint4(w[0], w[1], w[2], w[3]);
      }
    }
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    tc_fence_before();
    __syncthreads();
    if (tid == 0) {
      tc_fence_after();
      // dQ = dS K: A = dS K-major [q][key], B = K viewed MN-major ([d][key], d contiguous)
      constexpr uint32_t idQ = idesc_bf16(128, HD, false, true);
      const uint64_t dK_mn = mn_desc(base + B_OFF_K, 8192);
#pragma unroll
      for (int kb = 0; kb < 2; ++kb) {
        const uint64_t ds = kmajor_sw128_desc(base + B_OFF_S + kb * 16384);
#pragma unroll
        for (int k = 0; k < 4; ++k)
          tc_mma(tmem, ds + 2 * k, dK_mn + (uint64_t)(kb * 4 + k) * (2048 >> 4), idQ, (kb | k) != 0);
      }
      // dK = dS^T Q: A = dS viewed MN-major ([key][q]: two 64-key blocks 16 KB apart), B = Q MN-major
      constexpr uint32_t idK = idesc_bf16(128, HD, true, true);
      const uint64_t ds_mn = mn_desc(base + B_OFF_S, 16384), q_mn = mn_desc(base + B_OFF_Q, 8192);
#pragma unroll
      for (int k = 0; k < SEQ / 16; ++k)
        tc_mma(tmem + 64, ds_mn + (uint64_t)k * (2048 >> 4), q_mn + (uint64_t)k * (2048 >> 4), idK, k != 0);
      tc_commit(bar_a);
    }
    mbar_wait(bar_a, ph);  // dS consumed: Pd takes its place
    tc_fence_after();
    if (tid == 0 && more) load_qkv(it + gridDim.x);
#pragma unroll
    for (int c2 = 0; c2 < 2; ++c2) {
#pragma unroll
      for (int cc = 0; cc < 4; ++cc) {
        const int chunk = c2 * 4 + cc, j = c2 * 16 + cc * 4;
        *(uint4*)(srow + ((chunk ^ (row & 7)) << 4)) = make_uint4(pd[j], pd[j + 1], pd[j + 2], pd[j + 3]);
      }
    }
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    tc_fence_before();
    __syncthreads();
    if (tid == 0) {
      tc_fence_after();
      // dV = Pd^T dO: A = Pd viewed MN-major ([key][q]), B = dO MN-major ([d][q])
      constexpr uint32_t idV = idesc_bf16(128, HD, true, true);
      const uint64_t p_mn = mn_desc(base + B_OFF_S, 16384), do_mn = mn_desc(base + B_OFF_DO, 8192);
#pragma unroll
      for (int k = 0; k < SEQ / 16; ++k)
        tc_mma(tmem + 128, p_mn + (uint64_t)k * (2048 >> 4), do_mn + (uint64_t)k * (2048 >> 4), idV, k != 0);
      tc_commit(bar_v);
    }
    __nv_bfloat16* const out = a.dqkv + ((size_t)s * SEQ + row) * ld + h * HD + hf * 32;
    store_row32(out, lane_base + hf * 32);               // dq (query row), this half's 32 columns
    store_row32(out + a.Dm, lane_base + 64 + hf * 32);   // dk (key row)
    mbar_wait(bar_v, ph);
    tc_fence_after();
    if (tid == 0 && more) load_do(it + gridDim.x);
    store_row32(out + 2 * a.Dm, lane_base + 128 + hf * 32);  // dv (key row)
    tc_fence_before();
    __syncthreads();  // TMEM, the shared tiles and the exchange slots are free for the next item
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 0) {
    tc_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(B_TMEM_COLS) : "memory");
  }
}

}  // namespace attn_tc

int attn_fwd_tc_launch(const void* qkv, void* out, int n_seq, int Dm, int H, int seqs_per_est, int est_base, int L,
                       int layer, uint64_t seed, int64_t step, float p, const int64_t* step_dev, cudaStream_t s,
                       float* stats, uint32_t* mbits) {
  const int T = n_seq * attn_tc::SEQ;
  CUtensorMap mqk, mv;
  if (!make_map(&mqk, qkv, T, 3 * Dm, attn_tc::SEQ, 1, (int64_t)T * 3 * Dm) ||
      !make_map_mn(&mv, qkv, 3 * Dm, T, 1, (int64_t)T * 3 * Dm))
    return ERR_CUDA;
  static bool attr = false;
  if (!attr) {
    if (cudaFuncSetAttribute(attn_tc::attn_fwd_tc_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             attn_tc::SMEM) != cudaSuccess)
      return ERR_CUDA;
    attr = true;
  }
  attn_tc::Args a{(__nv_bfloat16*)out, Dm, H, seqs_per_est, est_base, L, layer, n_seq * H, seed, step, p, step_dev,
                  (float2*)stats, mbits};
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  const int grid = a.n_items < 4 * sms ? a.n_items : 4 * sms;
  attn_tc::attn_fwd_tc_kernel<<<grid, attn_tc::THREADS, attn_tc::SMEM, s>>>(mqk, mv, a);
  return cudaGetLastError() == cudaSuccess ? OK : ERR_CUDA;
}

int attn_bwd_tc_launch(const void* qkv, const void* dctx, void* dqkv, int n_seq, int Dm, int H, int seqs_per_est,
                       int est_base, int L, int layer, uint64_t seed, int64_t step, float p, const int64_t* step_dev,
                       cudaStream_t s, const float* stats, const uint32_t* mbits) {
  const int T = n_seq * attn_tc::SEQ;
  CUtensorMap mqk, mdo;
  if (!make_map(&mqk, qkv, T, 3 * Dm, attn_tc::SEQ, 1, (int64_t)T * 3 * Dm) ||
      !make_map(&mdo, dctx, T, Dm, attn_tc::SEQ, 1, (int64_t)T * Dm))
    return ERR_CUDA;
  static bool attr = false;
  if (!attr) {
    if (cudaFuncSetAttribute(attn_tc::attn_bwd_tc_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             attn_tc::B_SMEM) != cudaSuccess)
      return ERR_CUDA;
    attr = true;
  }
  attn_tc::BwdArgs a{(__nv_bfloat16*)dqkv, Dm, H, seqs_per_est, est_base, L, layer, n_seq * H, seed, step, p,
                     step_dev, (const float2*)stats, mbits};
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  const int grid = a.n_items < 2 * sms ? a.n_items : 2 * sms;
  attn_tc::attn_bwd_tc_kernel<<<grid, attn_tc::B_THREADS, attn_tc::B_SMEM, s>>>(mqk, mdo, a);
  return cudaGetLastError() == cudaSuccess ? OK : ERR_CUDA;
}

}  // namespace bt
