// bt_gemm.cu -- deterministic bf16 GEMM on the 5th-generation tensor cores.
//
// C[M][N] = A[M][K] * B[N][K]^T   (A, B bf16 K-contiguous -- the nn.Linear
// layout x @ W^T; C fp32 or bf16; fp32 accumulation in TMEM).
//
// SURVEY.md §8f row 2 / north_star "deterministic model kernels": the dense
// layers of the C3/C4 model stack (ResNet-18, BERT-base) run as tcgen05
// kernels whose result is a pure function of the inputs:
//   * every C tile is owned by exactly one CTA (no split-K, no atomics);
//   * its K loop runs in ascending order, 16-wide UMMA steps in ascending
//     order, accumulating into one TMEM tile;
// so the bits do not depend on the grid size, the SM count, the tile
// schedule or the GPU count -- the property the elastic step needs (an EST's
// gradients must not change when it moves to another GPU).
//
// Structure (one CTA per SM, persistent, static round-robin tile schedule):
//   warp 0   TMA producer: A/B k-blocks (128B swizzle) into a STAGES-deep
//            shared-memory ring (full/empty mbarriers);
//   warp 1   TMEM allocator + MMA issuer: one elected thread issues
//            tcgen05.mma.cta_group::1.kind::f16 (M=128, N=BN, K=16) and
//            tcgen05.commit's the stage back to the producer; two TMEM
//            accumulators (2 x BN fp32 columns) so the epilogue of tile i
//            overlaps the MMAs of tile i+1;
//   warps 2-5 epilogue: tcgen05.ld 32 lanes x 32 columns -> registers ->
//            st.global (row-contiguous 128 B per thread).
#include <cuda.h>
#include <cuda_bf16.h>
#include <cuda_runtime.h>
#include <stdint.h>
#include <stdlib.h>

#include "bt_common.cuh"
#include "bt_ffn.cuh"
#include "bt_tc.cuh"

namespace bt {
namespace gemm {

constexpr int BM = 128, BK = 64, UK = 16;  // tile M, k-block (128 B of bf16), UMMA K
#ifndef BT_EPI_WARPS
#define BT_EPI_WARPS 8
#endif
constexpr int EPI_WARPS = BT_EPI_WARPS;  // EPI_WARPS/4 per TMEM lane group, each draining a column slice
constexpr int EPI_SPLIT = EPI_WARPS / 4;
constexpr int THREADS = 64 + 32 * EPI_WARPS;

using namespace tc;  // bt_tc.cuh: mbarriers, TMA, tcgen05, UMMA descriptors

template <bool MN>
__device__ __forceinline__ uint64_t op_desc(uint32_t saddr) {
  return MN ? mnmajor_sw128_desc(saddr) : kmajor_sw128_desc(saddr);
}
template <bool MN>
constexpr uint64_t k_step() {  // descriptor increment per UMMA K step (16-byte units)
  return MN ? 2048 >> 4 : 32 >> 4;
}

// Instruction descriptor: D f32 [4,6)=1, A bf16 [7,10)=1, B bf16 [10,13)=1,
// both K-major, N>>3 at [17,23), M>>4 at [24,29).
// a_major [15] / b_major [16] = 1 for MN-major operands.
template <int BN, bool MN = false, bool BMN = false>
__device__ __forceinline__ constexpr uint32_t instr_desc() {
  return (1u << 4) | (1u << 7) | (1u << 10) | (MN ? (3u << 15) : 0u) | (BMN ? (1u << 16) : 0u) |
         ((uint32_t)(BN >> 3) << 17) | ((uint32_t)(BM >> 4) << 24);
}

// Tile t -> (m0, n0): groups of GROUP_M row-blocks walked column by column, so
// one wave of CTAs touches GROUP_M A row-blocks and a few B column-blocks
// (L2-resident) instead of streaming A once per B column.  The order only
// affects which CTA computes a tile, never a tile's bits.
constexpr int GROUP_M = 16;
template <int BN>
__device__ __forceinline__ void tile_coords_bn(int t, int mt, int nt, int* m0, int* n0) {
  const int per_group = GROUP_M * nt;
  const int g = t / per_group, r = t - g * per_group;
  const int gm = min(GROUP_M, mt - g * GROUP_M);  // rows in this (possibly short) last group
  *m0 = (g * GROUP_M + r % gm) * BM;
  *n0 = (r / gm) * BN;
}


__device__ __forceinline__ void tma_store_3d(const CUtensorMap* map, uint32_t src, int x, int y, int z) {
  asm volatile("cp.async.bulk.tensor.3d.global.shared::cta.bulk_group [%0, {%2, %3, %4}], [%1];" ::"l"(map), "r"(src),
               "r"(x), "r"(y), "r"(z)
               : "memory");
}
__device__ __forceinline__ void bulk_commit() { asm volatile("cp.async.bulk.commit_group;" ::: "memory"); }
__device__ __forceinline__ void bulk_wait_read1() { asm volatile("cp.async.bulk.wait_group.read 1;" ::: "memory"); }
__device__ __forceinline__ void bulk_wait_read0() { asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory"); }
// before re-staging a box: with NB boxes per warp the store that last used this box is NB chunks old
template <int NB>
__device__ __forceinline__ void bulk_wait_box() {
  if (NB == 1) bulk_wait_read0();
  else bulk_wait_read1();
}
__device__ __forceinline__ void bulk_wait0() { asm volatile("cp.async.bulk.wait_group 0;" ::: "memory"); }
__device__ __forceinline__ void fence_async_smem() { asm volatile("fence.proxy.async.shared::cta;" ::: "memory"); }

// Epilogue staging: each epilogue warp owns EPI_STAGE bytes of shared memory, holding one
// 32-row x 32-column box of C (and of the second output) in the TMA swizzled layout:
// fp32 rows of 128 B (SWIZZLE_128B: 16-byte chunk q of row r at q ^ (r & 7)), bf16 rows of
// 64 B (SWIZZLE_64B: chunk q at q ^ ((r >> 1) & 3)) -- conflict-free row-per-lane writes;
// one elected lane then issues a TMA bulk-tensor store (full 128-byte lines to L2/HBM).
constexpr int EPI_BOX = 4096;              // one 32 x 32 staging box (fp32, or two bf16 outputs)
constexpr int EPI_STAGE = 2 * EPI_BOX;     // double-buffered: chunk i stages in box i & 1
__device__ __forceinline__ void stage_f32(uint8_t* st, const float* f, int lane) {
#pragma unroll
  for (int q = 0; q < 8; ++q)
    *(float4*)(st + lane * 128 + ((q ^ (lane & 7)) << 4)) = make_float4(f[4 * q], f[4 * q + 1], f[4 * q + 2], f[4 * q + 3]);
}
__device__ __forceinline__ void stage_bf16(uint8_t* st, const float* f, int lane) {
#pragma unroll
  for (int q = 0; q < 4; ++q) {
    uint32_t w[4];
#pragma unroll
    for (int h = 0; h < 4; ++h) {
      const __nv_bfloat162 b2 = __floats2bfloat162_rn(f[q * 8 + 2 * h], f[q * 8 + 2 * h + 1]);
      w[h] = *(const uint32_t*)&b2;
    }
    *(uint4*)(st + lane * 64 + ((q ^ ((lane >> 1) & 3)) << 4)) = make_uint4(w[0], w[1], w[2], w[3]);
  }
}

// Column sums of a staged 32 x 32 bf16 box (SW64 layout, as the TMA store reads it): lane (h, cp) sums
// columns 2cp, 2cp+1 over the rows of parity h in ascending order (lanes 0-15 read one even row, lanes
// 16-31 the next odd row: the two 64-byte rows fill all 32 banks), then even + odd -- a fixed association
// of exactly the stored bf16 values.  out: 32 fp32 partials of this 32-row block.
__device__ __forceinline__ void colsum_box32(const uint8_t* st, int lane, float* out) {
  const int h = lane >> 4, cp = lane & 15, q = cp >> 2;
  ffn::f32x2 acc = ffn::pk2(0.f, 0.f);
#pragma unroll
  for (int i = 0; i < 16; ++i) {
    const int r = 2 * i + h;
    const uint32_t w = *(const uint32_t*)(st + r * 64 + ((q ^ ((r >> 1) & 3)) << 4) + (cp & 3) * 4);
    const float2 f = __bfloat1622float2(*(const __nv_bfloat162*)&w);
    acc = ffn::add2(acc, ffn::pk2(f.x, f.y));
  }
  const float2 a = ffn::upk2(acc);
  const float ox = __shfl_xor_sync(0xffffffffu, a.x, 16), oy = __shfl_xor_sync(0xffffffffu, a.y, 16);
  if (h == 0) *(float2*)(out + 2 * cp) = make_float2(__fadd_rn(a.x, ox), __fadd_rn(a.y, oy));
}

// One epilogue chunk: 32 consecutive fp32 accumulators of row `row` (lane = row - row0),
// columns [col, col+32) -- plain (fp32 / bf16), + bias, or an FFN element op fused in --
// staged in shared memory and stored by TMA at (col, row0, batch entry z).
template <bool OUT_BF16, int NB = 2>
__device__ __forceinline__ void epilogue_chunk(const uint32_t* v, size_t row, int col, int N, const GemmEpi& epi,
                                               uint8_t* st, int lane, const CUtensorMap* mc, const CUtensorMap* mc2,
                                               int row0, int z) {
  if (epi.kind == EPI_FFN_FWD) {
    // bias + GELU' (C) and dropout(GELU) (out2), produced and staged 8 columns at a time (few live
    // registers: the 16-epilogue-warp kernel has ~96 per thread)
    const int e = (int)(row / (size_t)epi.Te), tl = (int)(row - (size_t)e * epi.Te);
    const uint64_t sd = epi.p > 0.f ? derive3(ffn::TAG_FFN_DROP, epi.seed, (uint64_t)(epi.est_base + e)) : 0;
    const float keep = epi.p < 1.f ? 1.f / (1.f - epi.p) : 0.f;
    if (lane == 0) bulk_wait_box<NB>();  // the store that last used this box (two chunks ago) has read it
    __syncwarp();
#pragma unroll
    for (int q8 = 0; q8 < 4; ++q8) {
      const float4 b0 = *(const float4*)(epi.bias + col + 8 * q8), b1 = *(const float4*)(epi.bias + col + 8 * q8 + 4);
      const ffn::f32x2 bb[4] = {ffn::pk2(b0.x, b0.y), ffn::pk2(b0.z, b0.w), ffn::pk2(b1.x, b1.y),
                                ffn::pk2(b1.z, b1.w)};
      uint32_t wc[4], wo[4];
#pragma unroll
      for (int h = 0; h < 4; ++h) {  // packed pairs: the same operations, bit for bit, at half the issue count
        const int q = 8 * q8 + 2 * h;
        ffn::f32x2 g, d;
        ffn::gelu_and_grad2(ffn::add2(ffn::pk2(__uint_as_float(v[q]), __uint_as_float(v[q + 1])), bb[h]), &g, &d);
        if (epi.p > 0.f) {
          float m0, m1;
          ffn::drop_scale2(sd, epi.step, epi.Te, N, tl, col + q, epi.p, keep, &m0, &m1);
          g = ffn::mul2(g, ffn::pk2(m0, m1));
        }
        wc[h] = ffn::bf16x2_bits(d);
        wo[h] = ffn::bf16x2_bits(g);
      }
      const int off = lane * 64 + ((q8 ^ ((lane >> 1) & 3)) << 4);  // SW64 box layout
      *(uint4*)(st + off) = make_uint4(wc[0], wc[1], wc[2], wc[3]);
      *(uint4*)(st + EPI_BOX / 2 + off) = make_uint4(wo[0], wo[1], wo[2], wo[3]);
    }
    fence_async_smem();
    __syncwarp();
    if (lane == 0) {
      tma_store_3d(mc, su32(st), col, row0, z);
      tma_store_3d(mc2, su32(st + EPI_BOX / 2), col, row0, z);
      bulk_commit();
    }
    return;
  }
  if (epi.kind == EPI_FFN_BWD) {
    // C = acc * dropout_scale * gelu'(h): the aux box (32 rows x 32 bf16) staged in the second half of
    // this warp's staging box with coalesced loads, consumed and the output staged 8 columns at a time
    const int e = (int)(row / (size_t)epi.Te), tl = (int)(row - (size_t)e * epi.Te);
    const uint64_t sd = epi.p > 0.f ? derive3(ffn::TAG_FFN_DROP, epi.seed, (uint64_t)(epi.est_base + e)) : 0;
    const float keep = epi.p < 1.f ? 1.f / (1.f - epi.p) : 0.f;
    uint8_t* const ab = st + EPI_BOX / 2;
    if (lane == 0) bulk_wait_box<NB>();
    __syncwarp();
#pragma unroll
    for (int pass = 0; pass < 4; ++pass) {
      const int rr = pass * 8 + (lane >> 2), qq = lane & 3;
      const uint4 a4 = *(const uint4*)(epi.aux + ((size_t)row0 + rr) * N + col + qq * 8);
      *(uint4*)(ab + rr * 64 + ((qq ^ ((rr >> 1) & 3)) << 4)) = a4;
    }
    __syncwarp();
#pragma unroll
    for (int q8 = 0; q8 < 4; ++q8) {
      const int off = lane * 64 + ((q8 ^ ((lane >> 1) & 3)) << 4);
      const uint4 u = *(const uint4*)(ab + off);
      const __nv_bfloat162* h2 = (const __nv_bfloat162*)&u;
      uint32_t w[4];
#pragma unroll
      for (int k = 0; k < 4; ++k) {
        const float2 gp = __bfloat1622float2(h2[k]);
        const int q = 8 * q8 + 2 * k;
        ffn::f32x2 a = ffn::pk2(__uint_as_float(v[q]), __uint_as_float(v[q + 1]));
        if (epi.p > 0.f) {  // (acc * m) * gelu'; without dropout m = 1 and acc * 1 = acc exactly
          float m0, m1;
          ffn::drop_scale2(sd, epi.step, epi.Te, N, tl, col + q, epi.p, keep, &m0, &m1);
          a = ffn::mul2(a, ffn::pk2(m0, m1));
        }
        w[k] = ffn::bf16x2_bits(ffn::mul2(a, ffn::pk2(gp.x, gp.y)));
      }
      *(uint4*)(st + off) = make_uint4(w[0], w[1], w[2], w[3]);
    }
    fence_async_smem();
    __syncwarp();
    if (lane == 0) {
      tma_store_3d(mc, su32(st), col, row0, z);
      bulk_commit();
    }
    if (epi.colpart) colsum_box32(st, lane, epi.colpart + (size_t)(row0 >> 5) * N + col);
    return;
  }
  float f[32];
#pragma unroll
  for (int q = 0; q < 32; ++q) f[q] = __uint_as_float(v[q]);
  if (epi.kind == EPI_BIAS) {
#pragma unroll
    for (int q4 = 0; q4 < 8; ++q4) {
      const float4 bv = *(const float4*)(epi.bias + col + 4 * q4);
      f[4 * q4] += bv.x;
      f[4 * q4 + 1] += bv.y;
      f[4 * q4 + 2] += bv.z;
      f[4 * q4 + 3] += bv.w;
    }
  }
  if (lane == 0) bulk_wait_box<NB>();  // the store that last used this box (two chunks ago) has read it
  __syncwarp();
  if (OUT_BF16) {
    stage_bf16(st, f, lane);
  } else {
    stage_f32(st, f, lane);
  }
  fence_async_smem();
  __syncwarp();
  if (lane == 0) {
    tma_store_3d(mc, su32(st), col, row0, z);
    bulk_commit();
  }
}

// Implicit-GEMM convolution (TMA im2col mode).  The activation is NHWC [N][H][W][Ci] (Ci % 64 == 0);
// GEMM row / K index q of an operand is the output pixel (n, ho, wo) in row-major order; a K block
// (forward) or N block (weight gradient) of 64 is one filter tap (kh, kw) x 64 input channels, in the
// order (tap, channel) -- the explicit im2col's column order, so the tiles (and the bits) are the same.
// The tensor map's pixel box is [-p, (Wo-1)s - p] x [-p, (Ho-1)s - p] with traversal stride s, so a
// column of consecutive output pixels wraps rows and images exactly as the GEMM rows do; the load
// starts at input (wo*s - p, ho*s - p, n) and adds the tap offset (kw, kh).
struct ConvGeom {
  int Ho, Wo, s, p, KW, cblocks;  // cblocks = Ci / 64
  int rows_per_batch;             // output pixels per batch entry (weight gradient: one EST's pixels)
};
__device__ __forceinline__ void tma_load_im2col(uint32_t dst, const CUtensorMap* map, int c, int w, int h, int n,
                                                int ow, int oh, uint32_t bar) {
  asm volatile(
      "cp.async.bulk.tensor.4d.shared::cluster.global.im2col.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4, "
      "%5}], [%6], {%7, %8};" ::"r"(dst),
      "l"(map), "r"(c), "r"(w), "r"(h), "r"(n), "r"(bar), "h"((uint16_t)ow), "h"((uint16_t)oh)
      : "memory");
}
// im2col load of the 64 channels of tap `t`, channel block `cb`, for the column starting at output pixel q
__device__ __forceinline__ void conv_load(uint32_t dst, const CUtensorMap* map, const ConvGeom& g, int q, int t,
                                          int cb, uint32_t bar) {
  const int hw = g.Ho * g.Wo;
  const int n = q / hw, r = q - n * hw, ho = r / g.Wo, wo = r - ho * g.Wo;
  const int kh = t / g.KW, kw = t - kh * g.KW;
  tma_load_im2col(dst, map, cb * 64, wo * g.s - g.p, ho * g.s - g.p, n, kw, kh, bar);
}

constexpr int RB_KB = 9;  // resident-weight form (AIM 3): up to 9 k-blocks (K <= 576) of a BN = 64 B operand
template <int BN, int STAGES, int RB = 0>
struct Smem {
  static constexpr int A_BYTES = BM * BK * 2, B_BYTES = BN * BK * 2;
  static constexpr int STAGE = A_BYTES + (RB ? 0 : B_BYTES);  // RB: only A streams through the stages
  static constexpr int RES = STAGES * STAGE;                  // resident B: RB k-blocks
  static constexpr int EPI = RES + RB * B_BYTES;              // epilogue staging, EPI_STAGE per epilogue warp
  static constexpr int BAR = EPI + EPI_WARPS * EPI_STAGE;     // full[S], empty[S], tfull[2], tempty[2], bres, tmem addr
  static constexpr int TOTAL = BAR + (2 * STAGES + 5) * 8 + 16;
};

// AIM: 0 = tiled operands; 4 = tiled, A K-major and B MN-major (C = A.B with B stored [K][N]: the dX
// products read the weights as stored, no transposed copy); 1 = A is im2col(x) (forward convolution, K-major); 2 = B is im2col(x)
// (weight gradient dW = dz^T im2col(x), MN-major, K = output pixels of one batch entry); 3 = AIM 1 with
// the whole B operand (N <= 64, K <= 576: the filter) loaded once per CTA and kept resident in shared
// memory, so only the im2col A tiles stream (the same UMMAs in the same order: the same bits)
template <int BN, int STAGES, bool OUT_BF16, bool MN, int AIM = 0>
__global__ void __launch_bounds__(THREADS, 1)
    gemm_bf16_tn_kernel(const __grid_constant__ CUtensorMap map_a, const __grid_constant__ CUtensorMap map_b,
                        const __grid_constant__ CUtensorMap map_c, const __grid_constant__ CUtensorMap map_c2, int M,
                        int N, int K, int batch, const GemmEpi epi, const ConvGeom cg) {
  using L = Smem<BN, STAGES, AIM == 3 ? RB_KB : 0>;
  extern __shared__ uint8_t smem_raw[];
  const uint32_t raw = su32(smem_raw);
  const uint32_t base = (raw + 1023u) & ~1023u;  // SW128 tiles need 1024-byte alignment
  uint8_t* const gbase = smem_raw + (base - raw);
  const uint32_t bar0 = base + L::BAR;
  auto full = [&](int s) { return bar0 + 8u * s; };
  auto empty = [&](int s) { return bar0 + 8u * (STAGES + s); };
  auto tfull = [&](int a) { return bar0 + 8u * (2 * STAGES + a); };
  auto tempty = [&](int a) { return bar0 + 8u * (2 * STAGES + 2 + a); };
  const uint32_t bres = bar0 + 8u * (2 * STAGES + 4);  // AIM 3: the resident B operand landed
  uint32_t* const tmem_slot = (uint32_t*)(gbase + L::BAR + (2 * STAGES + 5) * 8);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int mt = (M + BM - 1) / BM, nt = (N + BN - 1) / BN, kb_n = (K + BK - 1) / BK;  // TMA zero-fills / clips edges
  const int per_batch = mt * nt;
  auto tile_coords = [&](int t, int mt_, int nt_, int* m0, int* n0) {  // t -> (batch entry, m0, n0)
    tile_coords_bn<BN>(t % per_batch, mt_, nt_, m0, n0);
  };
  const int tiles = per_batch * batch;

  if (warp == 0 && lane == 0) {
    asm volatile("prefetch.tensormap [%0];" ::"l"(&map_a) : "memory");
    asm volatile("prefetch.tensormap [%0];" ::"l"(&map_b) : "memory");
    for (int s = 0; s < STAGES; ++s) {
      mbar_init(full(s), 1);
      mbar_init(empty(s), 1);
    }
    for (int a = 0; a < 2; ++a) {
      mbar_init(tfull(a), 1);
      mbar_init(tempty(a), EPI_WARPS);  // one arrival per epilogue warp
    }
    mbar_init(bres, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == 1) {  // 2 x BN fp32 accumulator columns (power of two >= 32)
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(su32(tmem_slot)),
                 "r"(2 * BN)
                 : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;

  if (warp == 0) {
    // ---- TMA producer ------------------------------------------------------
    if (lane == 0) {
      int stage = 0;
      uint32_t phase = 0;
      if constexpr (AIM == 3) {  // the filter, once (one N tile, batch 1)
        mbar_arrive_expect_tx(bres, kb_n * L::B_BYTES);
        for (int kb = 0; kb < kb_n; ++kb) tma_load_3d(base + L::RES + kb * L::B_BYTES, &map_b, kb * BK, 0, 0, bres);
      }
      for (int t = blockIdx.x; t < tiles; t += gridDim.x) {
        int m0, n0;
        tile_coords(t, mt, nt, &m0, &n0);
        for (int kb = 0; kb < kb_n; ++kb) {
          mbar_wait(empty(stage), phase ^ 1u);
          const uint32_t sa = base + stage * L::STAGE, sb = sa + L::A_BYTES;
          mbar_arrive_expect_tx(full(stage), L::STAGE);
          if constexpr (AIM == 3) {
            const int tap = kb / cg.cblocks;
            conv_load(sa, &map_a, cg, m0, tap, kb - tap * cg.cblocks, full(stage));
          } else if constexpr (AIM == 1) {  // 128 output pixels x (tap, 64 channels); weights K-major
            const int tap = kb / cg.cblocks;
            conv_load(sa, &map_a, cg, m0, tap, kb - tap * cg.cblocks, full(stage));
            tma_load_3d(sb, &map_b, kb * BK, n0, t / per_batch, full(stage));
          } else if constexpr (AIM == 2) {  // dz MN-major; im2col columns of 64 pixels per 64-wide N block
#pragma unroll
            for (int j = 0; j < BM / 64; ++j)
              tma_load_3d(sa + j * MN_BLOCK_BYTES, &map_a, m0 + 64 * j, kb * BK, t / per_batch, full(stage));
            const int q = (t / per_batch) * cg.rows_per_batch + kb * BK;
#pragma unroll
            for (int j = 0; j < BN / 64; ++j) {
              const int nb = (n0 >> 6) + j, tap = nb / cg.cblocks;
              conv_load(sb + j * MN_BLOCK_BYTES, &map_b, cg, q, tap, nb - tap * cg.cblocks, full(stage));
            }
          } else if constexpr (MN) {  // [k][mn] operands: one 64 x 64 box per 64-wide MN block
#pragma unroll
            for (int j = 0; j < BM / 64; ++j)
              tma_load_3d(sa + j * MN_BLOCK_BYTES, &map_a, m0 + 64 * j, kb * BK, t / per_batch, full(stage));
#pragma unroll
            for (int j = 0; j < BN / 64; ++j)
              tma_load_3d(sb + j * MN_BLOCK_BYTES, &map_b, n0 + 64 * j, kb * BK, t / per_batch, full(stage));
          } else if constexpr (AIM == 4) {  // A K-major box; B [k][n]: one 64 x 64 box per 64-wide N block
            tma_load_3d(sa, &map_a, kb * BK, m0, t / per_batch, full(stage));
#pragma unroll
            for (int j = 0; j < BN / 64; ++j)
              tma_load_3d(sb + j * MN_BLOCK_BYTES, &map_b, n0 + 64 * j, kb * BK, t / per_batch, full(stage));
          } else {
            tma_load_3d(sa, &map_a, kb * BK, m0, t / per_batch, full(stage));
            tma_load_3d(sb, &map_b, kb * BK, n0, t / per_batch, full(stage));
          }
          if (++stage == STAGES) {
            stage = 0;
            phase ^= 1u;
          }
        }
      }
    }
  } else if (warp == 1) {
    // ---- MMA issuer --------------------------------------------------------
    if (lane == 0) {
      constexpr uint32_t idesc = instr_desc<BN, MN, AIM == 4>();
      constexpr bool BMJ = MN || AIM == 4;  // B operand MN-major
      int stage = 0;
      uint32_t phase = 0;
      int i = 0;
      if constexpr (AIM == 3) mbar_wait(bres, 0);
      for (int t = blockIdx.x; t < tiles; t += gridDim.x, ++i) {
        const int acc = i & 1;
        mbar_wait(tempty(acc), ((i >> 1) & 1) ^ 1u);  // the epilogue drained this accumulator
        tc_fence_after();
        const uint32_t d = tmem + (uint32_t)(acc * BN);
        for (int kb = 0; kb < kb_n; ++kb) {
          mbar_wait(full(stage), phase);
          tc_fence_after();
          const uint32_t sa = base + stage * L::STAGE;
          const uint32_t sb = AIM == 3 ? base + L::RES + kb * L::B_BYTES : sa + L::A_BYTES;
          const uint64_t da = op_desc<MN>(sa), db = op_desc<BMJ>(sb);
#pragma unroll
          for (int k = 0; k < BK / UK; ++k)  // K-major: +32 B inside the swizzled row; MN-major: +2 k groups
            tc_mma(d, da + k * k_step<MN>(), db + k * k_step<BMJ>(), idesc, (kb | k) != 0);
          tc_commit(empty(stage));  // frees the smem stage when these MMAs complete
          if (++stage == STAGES) {
            stage = 0;
            phase ^= 1u;
          }
        }
        tc_commit(tfull(acc));  // accumulator complete
      }
    }
  } else {
    // ---- epilogue: TMEM -> registers -> global -------------------------------
    const int lg = warp & 3;  // TMEM lane group this warp may access (lanes 32*lg ...)
    const int half = (warp - 2) >> 2;  // which column slice (of EPI_SPLIT)
    uint8_t* const est = gbase + L::EPI + (warp - 2) * EPI_STAGE;
    int chunk = 0;  // alternates the two staging boxes
    int i = 0;
    for (int t = blockIdx.x; t < tiles; t += gridDim.x, ++i) {
      const int acc = i & 1;
      int m0, n0;
      tile_coords(t, mt, nt, &m0, &n0);
      mbar_wait(tfull(acc), (i >> 1) & 1);
      tc_fence_after();
      const int row0 = m0 + lg * 32;  // this warp's 32 rows (lane = row - row0) within the batch entry
      const size_t row = (size_t)row0 + lane;
#pragma unroll 1
      constexpr int PER = BN / EPI_SPLIT < 32 ? 32 : BN / EPI_SPLIT;  // columns per epilogue warp (BN=64: 8 warps work)
      for (int cc = half * PER; cc < (half + 1) * PER && cc < BN; cc += 32) {
        uint32_t v[32];
        tmem_ld32(tmem + ((uint32_t)(lg * 32) << 16) + (uint32_t)(acc * BN + cc), v);
        tmem_ld_wait();
        epilogue_chunk<OUT_BF16>(v, row, n0 + cc, N, epi, est + (chunk++ & 1) * EPI_BOX, lane, &map_c, &map_c2, row0,
                                  t / per_batch);
      }
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(tempty(acc));
    }
    if (lane == 0) bulk_wait0();  // this warp's stores complete before the CTA exits
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 1) {
    tc_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(2 * BN) : "memory");
  }
}


// ---------------------------------------------------------------------------
// CTA-pair form (cta_group::2): a cluster of 2 CTAs on one TPC computes a
// 256 x 256 tile with M = 256 UMMAs issued by the leader.  Each CTA loads its
// 128 rows of A and 128 rows of B (half the operand traffic of two 1-CTA
// tiles); both CTAs' TMA bytes complete on the leader's full barrier; the
// leader's commits multicast to both CTAs' empty / accumulator barriers; each
// CTA drains its own 128 TMEM lanes.  Same per-element order as the 1-CTA
// kernel (one tile owner, ascending K), so the same determinism guarantee.
__device__ __forceinline__ uint32_t cluster_rank() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
  return r;
}
__device__ __forceinline__ void tma_load_3d_pair(uint32_t dst, const CUtensorMap* map, int x, int y, int z,
                                                 uint32_t leader_bar) {
  asm volatile(
      "cp.async.bulk.tensor.3d.cta_group::2.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, "
      "%3, %4}], [%5];" ::"r"(dst),
      "l"(map), "r"(x), "r"(y), "r"(z), "r"(leader_bar)
      : "memory");
}
__device__ __forceinline__ void conv_load_pair(uint32_t dst, const CUtensorMap* map, const ConvGeom& g, int q, int t,
                                               int cb, uint32_t leader_bar) {  // conv_load, bytes to the leader
  const int hw = g.Ho * g.Wo;
  const int n = q / hw, r = q - n * hw, ho = r / g.Wo, wo = r - ho * g.Wo;
  const int kh = t / g.KW, kw = t - kh * g.KW;
  asm volatile(
      "cp.async.bulk.tensor.4d.cta_group::2.shared::cluster.global.im2col.mbarrier::complete_tx::bytes [%0], [%1, {%2, "
      "%3, %4, %5}], [%6], {%7, %8};" ::"r"(dst),
      "l"(map), "r"(cb * 64), "r"(wo * g.s - g.p), "r"(ho * g.s - g.p), "r"(n), "r"(leader_bar), "h"((uint16_t)kw),
      "h"((uint16_t)kh)
      : "memory");
}
__device__ __forceinline__ void tc_mma_pair(uint32_t d_tmem, uint64_t adesc, uint64_t bdesc, uint32_t idesc, int acc) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::2.kind::f16 [%0], %1, %2, %3, p;\n\t}" ::"r"(d_tmem),
      "l"(adesc), "l"(bdesc), "r"(idesc), "r"(acc)
      : "memory");
}
__device__ __forceinline__ void tc_commit_pair(uint32_t bar) {  // arrive on this offset in both CTAs
  asm volatile(
      "tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;" ::"r"(bar),
      "h"((uint16_t)3)
      : "memory");
}
__device__ __forceinline__ void mbar_arrive_remote(uint32_t cluster_bar) {
  asm volatile("mbarrier.arrive.release.cluster.shared::cluster.b64 _, [%0];" ::"r"(cluster_bar) : "memory");
}
__device__ __forceinline__ uint32_t map_to_rank(uint32_t local, uint32_t rank) {
  uint32_t out;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(out) : "r"(local), "r"(rank));
  return out;
}

constexpr int PAIR_BN = 256, PAIR_M = 256;

template <int STAGES, int EW = EPI_WARPS, int NB = 2>
struct PairSmem {
  static constexpr int A_BYTES = BM * BK * 2, B_BYTES = (PAIR_BN / 2) * BK * 2;
  static constexpr int STAGE = A_BYTES + B_BYTES;
  static constexpr int EPI = STAGES * STAGE;
  static constexpr int BAR = EPI + EW * NB * EPI_BOX;
  static constexpr int TOTAL = BAR + (2 * STAGES + 4) * 8 + 16;
};

// EW epilogue warps (16 for ALU-heavy epilogues); AIM 1: A = im2col(x) K-major (the forward convolution);
// AIM 2: B = im2col(x) MN-major (the weight gradient)
template <int STAGES, bool OUT_BF16, bool MN, int EW = EPI_WARPS, int AIM = 0, int NB = 2>
__global__ void __launch_bounds__(64 + 32 * EW, 1)
    gemm_bf16_tn_pair_kernel(const __grid_constant__ CUtensorMap map_a, const __grid_constant__ CUtensorMap map_b,
                             const __grid_constant__ CUtensorMap map_c, const __grid_constant__ CUtensorMap map_c2,
                             int M, int N, int K, int batch, const GemmEpi epi, const ConvGeom cg) {
  using L = PairSmem<STAGES, EW, NB>;
  extern __shared__ uint8_t smem_raw[];
  const uint32_t raw = su32(smem_raw);
  const uint32_t base = (raw + 1023u) & ~1023u;
  uint8_t* const gbase = smem_raw + (base - raw);
  const uint32_t bar0 = base + L::BAR;
  auto full = [&](int s) { return bar0 + 8u * s; };
  auto empty = [&](int s) { return bar0 + 8u * (STAGES + s); };
  auto tfull = [&](int a) { return bar0 + 8u * (2 * STAGES + a); };
  auto tempty = [&](int a) { return bar0 + 8u * (2 * STAGES + 2 + a); };
  uint32_t* const tmem_slot = (uint32_t*)(gbase + L::BAR + (2 * STAGES + 4) * 8);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const uint32_t rank = cluster_rank();
  const bool leader = rank == 0;
  const int mt = M / PAIR_M, nt = N / PAIR_BN, kb_n = (K + BK - 1) / BK;
  const int per_batch = mt * nt;
  const int tiles = per_batch * batch;
  const int pair = blockIdx.x >> 1, pairs = gridDim.x >> 1;
  auto coords = [&](int t, int* m0, int* n0) {  // grouped raster, as the 1-CTA kernel
    t %= per_batch;
    constexpr int GM = GROUP_M / 2;
    const int per_group = GM * nt;
    const int g = t / per_group, r = t - g * per_group;
    const int gm = min(GM, mt - g * GM);
    *m0 = (g * GM + r % gm) * PAIR_M;
    *n0 = (r / gm) * PAIR_BN;
  };

  if (warp == 0 && lane == 0) {
    asm volatile("prefetch.tensormap [%0];" ::"l"(&map_a) : "memory");
    asm volatile("prefetch.tensormap [%0];" ::"l"(&map_b) : "memory");
    for (int s = 0; s < STAGES; ++s) {
      mbar_init(full(s), 1);   // leader: its expect_tx arrival; the bytes come from both CTAs
      mbar_init(empty(s), 1);  // each CTA: the leader's multicast commit
    }
    for (int a = 0; a < 2; ++a) {
      mbar_init(tfull(a), 1);
      mbar_init(tempty(a), 2 * EW);  // leader: every epilogue warp of both CTAs
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == 1) {
    asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(su32(tmem_slot)),
                 "r"(2 * PAIR_BN)
                 : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;" ::: "memory");
  }
  tc_fence_before();
  asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;

  if (warp == 0) {
    if (lane == 0) {  // ---- TMA producer (both CTAs: own A half, own B half) ----
      int stage = 0;
      uint32_t phase = 0;
      for (int t = pair; t < tiles; t += pairs) {
        int m0, n0;
        coords(t, &m0, &n0);
        for (int kb = 0; kb < kb_n; ++kb) {
          mbar_wait(empty(stage), phase ^ 1u);
          const uint32_t sa = base + stage * L::STAGE, sb = sa + L::A_BYTES;
          const uint32_t lb = full(stage) & 0xFEFFFFFFu;  // the leader CTA's barrier
          if (leader) mbar_arrive_expect_tx(full(stage), 2 * L::STAGE);
          if constexpr (MN) {
#pragma unroll
            for (int j = 0; j < BM / 64; ++j)
              tma_load_3d_pair(sa + j * MN_BLOCK_BYTES, &map_a, m0 + (int)rank * BM + 64 * j, kb * BK, t / per_batch,
                               lb);
            if constexpr (AIM == 2) {  // 64-pixel x 64-channel im2col blocks of this CTA's N half
              const int q = (t / per_batch) * cg.rows_per_batch + kb * BK;
#pragma unroll
              for (int j = 0; j < PAIR_BN / 128; ++j) {
                const int nb = ((n0 + (int)rank * (PAIR_BN / 2)) >> 6) + j, tap = nb / cg.cblocks;
                conv_load_pair(sb + j * MN_BLOCK_BYTES, &map_b, cg, q, tap, nb - tap * cg.cblocks, lb);
              }
            } else {
#pragma unroll
              for (int j = 0; j < PAIR_BN / 128; ++j)
                tma_load_3d_pair(sb + j * MN_BLOCK_BYTES, &map_b, n0 + (int)rank * (PAIR_BN / 2) + 64 * j, kb * BK,
                                 t / per_batch, lb);
            }
          } else {
            if constexpr (AIM == 1) {  // this CTA's 128 output pixels x (tap, 64 channels)
              const int tap = kb / cg.cblocks;
              conv_load_pair(sa, &map_a, cg, m0 + (int)rank * BM, tap, kb - tap * cg.cblocks, lb);
            } else {
              tma_load_3d_pair(sa, &map_a, kb * BK, m0 + (int)rank * BM, t / per_batch, lb);
            }
            if constexpr (AIM == 4) {  // B [k][n]: this CTA's N half as 64 x 64 boxes
#pragma unroll
              for (int j = 0; j < PAIR_BN / 128; ++j)
                tma_load_3d_pair(sb + j * MN_BLOCK_BYTES, &map_b, n0 + (int)rank * (PAIR_BN / 2) + 64 * j, kb * BK,
                                 t / per_batch, lb);
            } else {
              tma_load_3d_pair(sb, &map_b, kb * BK, n0 + (int)rank * (PAIR_BN / 2), t / per_batch, lb);
            }
          }
          if (++stage == STAGES) {
            stage = 0;
            phase ^= 1u;
          }
        }
      }
    }
  } else if (warp == 1) {
    if (leader && lane == 0) {  // ---- MMA issuer (leader only) ----
      constexpr uint32_t idesc = (1u << 4) | (1u << 7) | (1u << 10) | (MN ? (3u << 15) : 0u) |
                                 (AIM == 4 ? (1u << 16) : 0u) | ((uint32_t)(PAIR_BN >> 3) << 17) |
                                 ((uint32_t)(PAIR_M >> 4) << 24);
      constexpr bool BMJ = MN || AIM == 4;  // B operand MN-major
      int stage = 0;
      uint32_t phase = 0;
      int i = 0;
      for (int t = pair; t < tiles; t += pairs, ++i) {
        const int acc = i & 1;
        mbar_wait(tempty(acc), ((i >> 1) & 1) ^ 1u);
        tc_fence_after();
        const uint32_t d = tmem + (uint32_t)(acc * PAIR_BN);
        for (int kb = 0; kb < kb_n; ++kb) {
          mbar_wait(full(stage), phase);
          tc_fence_after();
          const uint32_t sa = base + stage * L::STAGE, sb = sa + L::A_BYTES;
          const uint64_t da = op_desc<MN>(sa), db = op_desc<BMJ>(sb);
#pragma unroll
          for (int k = 0; k < BK / UK; ++k)
            tc_mma_pair(d, da + k * k_step<MN>(), db + k * k_step<BMJ>(), idesc, (kb | k) != 0);
          tc_commit_pair(empty(stage));
          if (++stage == STAGES) {
            stage = 0;
            phase ^= 1u;
          }
        }
        tc_commit_pair(tfull(acc));
      }
    }
  } else {  // ---- epilogue (both CTAs: own 128 rows) ----
    const int lg = warp & 3;
    const int half = (warp - 2) >> 2;
    uint8_t* const est = gbase + L::EPI + (warp - 2) * NB * EPI_BOX;
    int chunk = 0;
    const uint32_t leader_tempty0 = map_to_rank(tempty(0), 0), leader_tempty1 = map_to_rank(tempty(1), 0);
    const int c_lo = half * (PAIR_BN / (EW / 4)), c_hi = c_lo + PAIR_BN / (EW / 4);
    int i = 0;
    for (int t = pair; t < tiles; t += pairs, ++i) {
      const int acc = i & 1;
      int m0, n0;
      coords(t, &m0, &n0);
      mbar_wait(tfull(acc), (i >> 1) & 1);
      tc_fence_after();
      const int row0 = m0 + (int)rank * BM + lg * 32;
      const size_t row = (size_t)row0 + lane;
#pragma unroll 1
      for (int cc = c_lo; cc < c_hi; cc += 32) {
        uint32_t v[32];
        tmem_ld32(tmem + ((uint32_t)(lg * 32) << 16) + (uint32_t)(acc * PAIR_BN + cc), v);
        tmem_ld_wait();
        epilogue_chunk<OUT_BF16, NB>(v, row, n0 + cc, N, epi, est + (NB == 2 ? (chunk++ & 1) : 0) * EPI_BOX, lane,
                                      &map_c, &map_c2, row0, t / per_batch);
      }
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive_remote(acc ? leader_tempty1 : leader_tempty0);
    }
    if (lane == 0) bulk_wait0();
  }
  tc_fence_before();
  __syncthreads();
  asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
  if (warp == 1) {
    tc_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(2 * PAIR_BN) : "memory");
  }
}


// ---------------------------------------------------------------------------
// Halo form of the 3x3 / stride-1 / pad-1 convolution with 64 input channels and the filter resident
// (Co <= 64): a 128-pixel tile is 128/W whole output rows of one image, and every tap's A operand is a
// 128-row view of one of three halo boxes {64 ch, W px starting at kw-1, 128/W+2 rows starting at
// ho0-1} (TMA zero-fills the padding).  The kh taps are the views at row offsets kh*W (multiples of
// 1024 bytes, so the SW128 pattern is unchanged): 3 boxes per tile instead of 9 im2col boxes, while
// the UMMAs are exactly the im2col path's (tap order (kh, kw), the same rows, the same filter blocks):
// the same bits.  Two tiles of halo boxes in flight; the epilogue stores rows straight from registers
// (no staging), which is what leaves room for the resident filter.
constexpr int HALO_THREADS = 64 + 256;
__device__ __forceinline__ uint32_t pack_bf16(float lo, float hi) {
  const __nv_bfloat162 b2 = __floats2bfloat162_rn(lo, hi);
  return *(const uint32_t*)&b2;
}
template <int W>
struct HaloSmem {
  static constexpr int ROWS = BM / W + 2;                       // halo rows per box
  static constexpr int BOX = ROWS * W * 128;                    // one kw box (64 channels x 2 bytes per pixel)
  static constexpr int SLOT = 3 * BOX;                          // one tile's three boxes
  static constexpr int RES = 2 * SLOT;                          // the resident filter: 9 k-blocks x 64 x 64
  static constexpr int BAR = RES + 9 * 8192;                    // afull[2], aempty[2], bres, tfull[2], tempty[2]
  static constexpr int TOTAL = BAR + 9 * 8 + 16;
};
__device__ __forceinline__ void tma_load_4d_tile(uint32_t dst, const CUtensorMap* map, int c0, int c1, int c2, int c3,
                                                 uint32_t bar) {
  asm volatile(
      "cp.async.bulk.tensor.4d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4, %5}], "
      "[%6];" ::"r"(dst),
      "l"(map), "r"(c0), "r"(c1), "r"(c2), "r"(c3), "r"(bar)
      : "memory");
}
template <int W, bool OUT_BF16>
__global__ void __launch_bounds__(HALO_THREADS, 1)
    conv_halo_kernel(const __grid_constant__ CUtensorMap map_x, const __grid_constant__ CUtensorMap map_w,
                     void* __restrict__ out, int M, int Co, int H) {
  using L = HaloSmem<W>;
  extern __shared__ uint8_t smem_raw[];
  const uint32_t raw = su32(smem_raw), base = (raw + 1023u) & ~1023u;
  uint8_t* const gbase = smem_raw + (base - raw);
  const uint32_t bar0 = base + L::BAR;
  auto afull = [&](int i) { return bar0 + 8u * i; };
  auto aempty = [&](int i) { return bar0 + 8u * (2 + i); };
  const uint32_t bres = bar0 + 32u;
  auto tfull = [&](int i) { return bar0 + 8u * (5 + i); };
  auto tempty = [&](int i) { return bar0 + 8u * (7 + i); };
  uint32_t* const tmem_slot = (uint32_t*)(gbase + L::BAR + 9 * 8);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int tiles = (M + BM - 1) / BM, tpi = (H * W) / BM;  // tiles per image
  if (warp == 0 && lane == 0) {
    asm volatile("prefetch.tensormap [%0];" ::"l"(&map_x) : "memory");
    asm volatile("prefetch.tensormap [%0];" ::"l"(&map_w) : "memory");
    for (int i = 0; i < 2; ++i) {
      mbar_init(afull(i), 1);
      mbar_init(aempty(i), 1);
      mbar_init(tfull(i), 1);
      mbar_init(tempty(i), 8);  // one arrival per epilogue warp
    }
    mbar_init(bres, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == 1) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(su32(tmem_slot)), "r"(128)
                 : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;
  if (warp == 0) {
    if (lane == 0) {  // ---- TMA producer: the filter once, then three halo boxes per tile
      mbar_arrive_expect_tx(bres, 9 * 8192);
      for (int kb = 0; kb < 9; ++kb) tma_load_3d(base + L::RES + kb * 8192, &map_w, kb * BK, 0, 0, bres);
      int i = 0;
      for (int t = blockIdx.x; t < tiles; t += gridDim.x, ++i) {
        const int sl = i & 1;
        mbar_wait(aempty(sl), ((i >> 1) & 1) ^ 1u);
        const int n = t / tpi, ho0 = (t - n * tpi) * (BM / W);
        mbar_arrive_expect_tx(afull(sl), L::SLOT);
        for (int kw = 0; kw < 3; ++kw)
          tma_load_4d_tile(base + sl * L::SLOT + kw * L::BOX, &map_x, 0, kw - 1, ho0 - 1, n, afull(sl));
      }
    }
  } else if (warp == 1) {
    if (lane == 0) {  // ---- MMA issuer: the im2col path's UMMA sequence, A from the halo views
      constexpr uint32_t idesc = idesc_bf16(BM, 64, false, false);
      mbar_wait(bres, 0);
      int i = 0;
      for (int t = blockIdx.x; t < tiles; t += gridDim.x, ++i) {
        const int sl = i & 1, acc = i & 1;
        mbar_wait(tempty(acc), ((i >> 1) & 1) ^ 1u);
        mbar_wait(afull(sl), (i >> 1) & 1);
        tc_fence_after();
        const uint32_t d = tmem + (uint32_t)(acc * 64);
        for (int kb = 0; kb < 9; ++kb) {
          const int kh = kb / 3, kw = kb - kh * 3;
          const uint64_t da = kmajor_sw128_desc(base + sl * L::SLOT + kw * L::BOX + kh * W * 128);
          const uint64_t db = kmajor_sw128_desc(base + L::RES + kb * 8192);
#pragma unroll
          for (int k = 0; k < BK / UK; ++k) tc_mma(d, da + 2 * k, db + 2 * k, idesc, (kb | k) != 0);
        }
        tc_commit(aempty(sl));
        tc_commit(tfull(acc));
      }
    }
  } else {  // ---- epilogue: 8 warps = 4 TMEM lane groups x 2 column halves; rows stored from registers
    const int lg = warp & 3, half = (warp - 2) >> 2;  // a warp may only read TMEM lanes 32*(warp % 4)..
    int i = 0;
    for (int t = blockIdx.x; t < tiles; t += gridDim.x, ++i) {
      const int acc = i & 1;
      mbar_wait(tfull(acc), (i >> 1) & 1);
      tc_fence_after();
      const int row = t * BM + lg * 32 + lane, c0 = half * 32;
      uint32_t v[32];
      tmem_ld32(tmem + ((uint32_t)(lg * 32) << 16) + (uint32_t)(acc * 64 + c0), v);
      tmem_ld_wait();
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(tempty(acc));
      if (row < M && c0 < Co) {
        if constexpr (OUT_BF16) {
          uint4* o = (uint4*)((__nv_bfloat16*)out + (size_t)row * Co + c0);
          const int nq = min(4, (Co - c0) / 8);
          for (int q = 0; q < nq; ++q) {
            uint4 u;
            u.x = pack_bf16(__uint_as_float(v[8 * q]), __uint_as_float(v[8 * q + 1]));
            u.y = pack_bf16(__uint_as_float(v[8 * q + 2]), __uint_as_float(v[8 * q + 3]));
            u.z = pack_bf16(__uint_as_float(v[8 * q + 4]), __uint_as_float(v[8 * q + 5]));
            u.w = pack_bf16(__uint_as_float(v[8 * q + 6]), __uint_as_float(v[8 * q + 7]));
            o[q] = u;
          }
        } else {
          float4* o = (float4*)((float*)out + (size_t)row * Co + c0);
          const int nq = min(8, (Co - c0) / 4);
          for (int q = 0; q < nq; ++q)
            o[q] = make_float4(__uint_as_float(v[4 * q]), __uint_as_float(v[4 * q + 1]), __uint_as_float(v[4 * q + 2]),
                               __uint_as_float(v[4 * q + 3]));
        }
      }
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 1) {
    tc_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(128) : "memory");
  }
}

// Weight gradient of the 3x3 / stride-1 / pad-1 convolution with 64 or 128 input and output channels
// at W = 32 / 16 (ResNet layers 1 and 2) by halo boxes instead of im2col loads.  dW_z[co][(kh, kw, ci)] =
// sum_pixels dz[pix][co] x[pix + (kh-1, kw-1)][ci] over batch entry z's pixels (an EST's pinned split).
// A tile is (z, kw, 64-channel block cb): the MMA's B operand for the three kh taps is ONE MN-major view
// of N = 192 over a {64 ch, W px from kw-1, 64/W + 2 rows from h0-1} halo box -- the kh views are W pixel
// rows (W * 128 bytes, a multiple of 1 KB) apart, a uniform distance between 64-wide N blocks, so one UMMA
// (M 128, N 192, K 16) per k-step covers the three taps.  Per 64-pixel k-block a tile loads the dz box
// (8 KB per 64 output channels) and one halo box (8 + 16 KB / W... 16 KB at W = 32, 12 KB at W = 16);
// the im2col form loaded a 16 KB dz box per 128-column tile and 8 KB per (tap, channel block).  dz is
// the A operand with M = 128 (with 64 output channels rows 64-127 are a zero block written once per
// stage, as the im2col form's zero-filled half), K ascending in 16-wide steps as there: the same products
// in the same order per output element, the same bits (tests/test_gpu_resnet.py).
constexpr int WGH_THREADS = 64 + 256, WGH_STAGES = 6, WGH_N = 192;
template <int W>
struct WghSmem {
  static constexpr int ROWS = BK / W + 2;        // halo rows per box
  static constexpr int A = 2 * MN_BLOCK_BYTES;  // dz: M blocks 0 / 1 (zero when Co = 64)
  static constexpr int B = ROWS * W * 128;      // one (kw, channel block) box: ROWS x W px x 64 ch bf16
  static constexpr int STAGE = A + B;
  static constexpr int BAR = WGH_STAGES * STAGE;  // full[S], empty[S], tfull[2], tempty[2], tmem slot
  static constexpr int TOTAL = BAR + (2 * WGH_STAGES + 4) * 8 + 16;
};
__device__ __forceinline__ uint64_t mn_desc_lbo(uint32_t saddr, uint32_t lbo) {
  return (uint64_t)((saddr & 0x3FFFF) >> 4) | ((uint64_t)(lbo >> 4) << 16) | ((uint64_t)(1024 >> 4) << 32) |
         ((uint64_t)1 << 46) | ((uint64_t)2 << 61);
}
template <int W>
__global__ void __launch_bounds__(WGH_THREADS, 1)
    conv_wgrad_halo_kernel(const __grid_constant__ CUtensorMap map_dz, const __grid_constant__ CUtensorMap map_x,
                           float* __restrict__ out, int batch, int rpb, int H, int64_t sc, int Ci, int Co) {
  using L = WghSmem<W>;
  extern __shared__ uint8_t smem_raw[];
  const uint32_t raw = su32(smem_raw), base = (raw + 1023u) & ~1023u;
  uint8_t* const gbase = smem_raw + (base - raw);
  const uint32_t bar0 = base + L::BAR;
  auto full = [&](int st) { return bar0 + 8u * st; };
  auto empty = [&](int st) { return bar0 + 8u * (WGH_STAGES + st); };
  auto tfull = [&](int a) { return bar0 + 8u * (2 * WGH_STAGES + a); };
  auto tempty = [&](int a) { return bar0 + 8u * (2 * WGH_STAGES + 2 + a); };
  uint32_t* const tmem_slot = (uint32_t*)(gbase + L::BAR + (2 * WGH_STAGES + 4) * 8);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int cbn = Ci / 64, mbn = Co / 64, K = 9 * Ci;
  const int tiles = batch * 3 * cbn, kbn = rpb / BK;
  if (warp == 0 && lane == 0) {
    asm volatile("prefetch.tensormap [%0];" ::"l"(&map_dz) : "memory");
    asm volatile("prefetch.tensormap [%0];" ::"l"(&map_x) : "memory");
    for (int st = 0; st < WGH_STAGES; ++st) {
      mbar_init(full(st), 1);
      mbar_init(empty(st), 1);
    }
    for (int a = 0; a < 2; ++a) {
      mbar_init(tfull(a), 1);
      mbar_init(tempty(a), 8);  // one arrival per epilogue warp
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == 1) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(su32(tmem_slot)), "r"(512)
                 : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
  }
  if (warp >= 2 && mbn == 1) {  // 64 output channels: the A operand's second M block is zero in every stage
    for (int st = 0; st < WGH_STAGES; ++st) {
      uint4* zb = (uint4*)(gbase + st * L::STAGE + MN_BLOCK_BYTES);
      for (int i = threadIdx.x - 64; i < MN_BLOCK_BYTES / 16; i += 256) zb[i] = make_uint4(0, 0, 0, 0);
    }
    fence_async_smem();
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;
  if (warp == 0) {
    if (lane == 0) {  // ---- TMA producer: per k-block the dz box(es) and the (kw, channel block) halo box
      int stage = 0;
      uint32_t phase = 0;
      for (int t = blockIdx.x; t < tiles; t += gridDim.x) {
        const int z = t / (3 * cbn), r = t - z * 3 * cbn, kw = r / cbn, cb = r - kw * cbn;
        for (int kb = 0; kb < kbn; ++kb) {
          mbar_wait(empty(stage), phase ^ 1u);
          const uint32_t sa = base + stage * L::STAGE, sb = sa + L::A;
          mbar_arrive_expect_tx(full(stage), mbn * MN_BLOCK_BYTES + L::B);
          for (int j = 0; j < mbn; ++j) tma_load_3d(sa + j * MN_BLOCK_BYTES, &map_dz, 64 * j, kb * BK, z, full(stage));
          const int q0 = z * rpb + kb * BK, n = q0 / (H * W), h0 = (q0 - n * H * W) / W;
          tma_load_4d_tile(sb, &map_x, cb * 64, kw - 1, h0 - 1, n, full(stage));
          if (++stage == WGH_STAGES) {
            stage = 0;
            phase ^= 1u;
          }
        }
      }
    }
  } else if (warp == 1) {
    if (lane == 0) {  // ---- MMA issuer: one M 128 x N 192 UMMA per 16-pixel k-step (the three kh taps)
      constexpr uint32_t idesc = idesc_bf16(BM, WGH_N, true, true);
      int stage = 0;
      uint32_t phase = 0;
      int i = 0;
      for (int t = blockIdx.x; t < tiles; t += gridDim.x, ++i) {
        const int acc = i & 1;
        mbar_wait(tempty(acc), ((i >> 1) & 1) ^ 1u);
        tc_fence_after();
        const uint32_t d = tmem + (uint32_t)(acc * 256);
        for (int kb = 0; kb < kbn; ++kb) {
          mbar_wait(full(stage), phase);
          tc_fence_after();
          const uint32_t sa = base + stage * L::STAGE, sb = sa + L::A;
          const uint64_t da = mn_desc_lbo(sa, MN_BLOCK_BYTES), db = mn_desc_lbo(sb, W * 128);
#pragma unroll
          for (int k = 0; k < BK / UK; ++k)
            tc_mma(d, da + (uint64_t)k * (2048 >> 4), db + (uint64_t)k * (2048 >> 4), idesc, (kb | k) != 0);
          tc_commit(empty(stage));
          if (++stage == WGH_STAGES) {
            stage = 0;
            phase ^= 1u;
          }
        }
        tc_commit(tfull(acc));
      }
    }
  } else {  // ---- epilogue: TMEM lane = output channel; 192 columns = (kh, ci of block cb)
    const int lg = warp & 3, half = (warp - 2) >> 2;
    int i = 0;
    for (int t = blockIdx.x; t < tiles; t += gridDim.x, ++i) {
      const int acc = i & 1, z = t / (3 * cbn), r = t - z * 3 * cbn, kw = r / cbn, cb = r - kw * cbn;
      mbar_wait(tfull(acc), (i >> 1) & 1);
      tc_fence_after();
      if (lg < 2 * mbn) {
        const int co = lg * 32 + lane;
        float* const orow = out + (size_t)z * sc + (size_t)co * K;
#pragma unroll 1
        for (int cc = 0; cc < 3; ++cc) {
          const int col = half * 96 + cc * 32, kh = col >> 6, ci0 = col & 63;
          uint32_t v[32];
          tmem_ld32(tmem + ((uint32_t)(lg * 32) << 16) + (uint32_t)(acc * 256 + col), v);
          tmem_ld_wait();
          float4* o = (float4*)(orow + (kh * 3 + kw) * Ci + cb * 64 + ci0);
#pragma unroll
          for (int q = 0; q < 8; ++q)
            o[q] = make_float4(__uint_as_float(v[4 * q]), __uint_as_float(v[4 * q + 1]), __uint_as_float(v[4 * q + 2]),
                               __uint_as_float(v[4 * q + 3]));
        }
      }
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(tempty(acc));
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 1) {
    tc_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(512) : "memory");
  }
}

}  // namespace gemm

// ---------------------------------------------------------------- launcher
typedef CUresult (*PFN_encodeTiled)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                    const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                                    CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

static PFN_encodeTiled encode_fn() {
  static PFN_encodeTiled fn = nullptr;
  if (!fn) {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = (PFN_encodeTiled)p;
  }
  return fn;
}

// [batch][rows][K] bf16, K contiguous, batch entries `bstride` elements apart;
// box = 64 (128 B) x box_rows x 1, 128-byte swizzle
bool make_map(CUtensorMap* map, const void* ptr, int rows, int K, int box_rows, int batch, int64_t bstride) {
  PFN_encodeTiled enc = encode_fn();
  if (!enc) return false;
  const cuuint64_t dims[3] = {(cuuint64_t)K, (cuuint64_t)rows, (cuuint64_t)batch};
  const cuuint64_t strides[2] = {(cuuint64_t)K * 2, (cuuint64_t)bstride * 2};
  const cuuint32_t box[3] = {(cuuint32_t)gemm::BK, (cuuint32_t)box_rows, 1};
  const cuuint32_t estr[3] = {1, 1, 1};
  return enc(map, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 3, const_cast<void*>(ptr), dims, strides, box, estr,
             CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
             CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

// C [batch][rows][cols] (fp32 or bf16), entries `bstride` elements apart; box = 32 x 32 x 1 --
// the epilogue's staging box (fp32: 128-byte rows, SWIZZLE_128B; bf16: 64-byte rows, SWIZZLE_64B)
static bool make_store_map(CUtensorMap* map, const void* ptr, int rows, int cols, int batch, int64_t bstride,
                           bool bf16) {
  PFN_encodeTiled enc = encode_fn();
  if (!enc) return false;
  const int eb = bf16 ? 2 : 4;
  const cuuint64_t dims[3] = {(cuuint64_t)cols, (cuuint64_t)rows, (cuuint64_t)batch};
  const cuuint64_t strides[2] = {(cuuint64_t)cols * eb, (cuuint64_t)bstride * eb};
  const cuuint32_t box[3] = {32, 32, 1};
  const cuuint32_t estr[3] = {1, 1, 1};
  return enc(map, bf16 ? CU_TENSOR_MAP_DATA_TYPE_BFLOAT16 : CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 3, const_cast<void*>(ptr),
             dims, strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
             bf16 ? CU_TENSOR_MAP_SWIZZLE_64B : CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_NONE,
             CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

// MN-major operand: stored [batch][K][rows] (rows contiguous); box = 64 (128 B) x 64 k-rows x 1
bool make_map_mn(CUtensorMap* map, const void* ptr, int rows, int K, int batch, int64_t bstride) {
  PFN_encodeTiled enc = encode_fn();
  if (!enc) return false;
  const cuuint64_t dims[3] = {(cuuint64_t)rows, (cuuint64_t)K, (cuuint64_t)batch};
  const cuuint64_t strides[2] = {(cuuint64_t)rows * 2, (cuuint64_t)bstride * 2};
  const cuuint32_t box[3] = {64, (cuuint32_t)gemm::BK, 1};
  const cuuint32_t estr[3] = {1, 1, 1};
  return enc(map, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 3, const_cast<void*>(ptr), dims, strides, box, estr,
             CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
             CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

// NHWC activation [N][H][W][C] for the im2col loads: `pixels` output pixels x 64 channels per load
static bool make_im2col_map(CUtensorMap* map, const void* x, int N, int H, int W, int C, const gemm::ConvGeom& g,
                            int pixels) {
  typedef CUresult (*PFN_encodeIm2col)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                       const cuuint64_t*, const int*, const int*, cuuint32_t, cuuint32_t,
                                       const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle,
                                       CUtensorMapL2promotion, CUtensorMapFloatOOBfill);
  static PFN_encodeIm2col enc = nullptr;
  if (!enc) {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeIm2col", &p, cudaEnableDefault, &q) != cudaSuccess ||
        q != cudaDriverEntryPointSuccess)
      return false;
    enc = (PFN_encodeIm2col)p;
  }
  const cuuint64_t dims[4] = {(cuuint64_t)C, (cuuint64_t)W, (cuuint64_t)H, (cuuint64_t)N};
  const cuuint64_t strides[3] = {(cuuint64_t)C * 2, (cuuint64_t)W * C * 2, (cuuint64_t)H * W * C * 2};
  const int lower[2] = {-g.p, -g.p};
  const int upper[2] = {(g.Wo - 1) * g.s - g.p - (W - 1), (g.Ho - 1) * g.s - g.p - (H - 1)};
  const cuuint32_t estr[4] = {1, (cuuint32_t)g.s, (cuuint32_t)g.s, 1};
  return enc(map, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 4, const_cast<void*>(x), dims, strides, lower, upper, 64,
             (cuuint32_t)pixels, estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
             CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

// the halo form's activation map: [N][H][W][64] bf16, box {64, W, 128/W + 2, 1}, SW128, zero fill
static bool make_halo_map(CUtensorMap* map, const void* x, int N, int H, int W) {
  PFN_encodeTiled enc = encode_fn();
  if (!enc) return false;
  const cuuint64_t dims[4] = {64, (cuuint64_t)W, (cuuint64_t)H, (cuuint64_t)N};
  const cuuint64_t strides[3] = {128, (cuuint64_t)W * 128, (cuuint64_t)H * W * 128};
  const cuuint32_t box[4] = {64, (cuuint32_t)W, (cuuint32_t)(gemm::BM / W + 2), 1};
  const cuuint32_t estr[4] = {1, 1, 1, 1};
  return enc(map, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 4, const_cast<void*>(x), dims, strides, box, estr,
             CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
             CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}
// the weight-gradient halo map: [N][H][W][C] bf16, box {64 ch, W px, 64/W + 2 rows, 1} (the k-block's
// output rows + the halo rows)
static bool make_wg_halo_map(CUtensorMap* map, const void* x, int N, int H, int W, int C) {
  PFN_encodeTiled enc = encode_fn();
  if (!enc) return false;
  const cuuint64_t dims[4] = {(cuuint64_t)C, (cuuint64_t)W, (cuuint64_t)H, (cuuint64_t)N};
  const cuuint64_t strides[3] = {(cuuint64_t)C * 2, (cuuint64_t)W * C * 2, (cuuint64_t)H * W * C * 2};
  const cuuint32_t box[4] = {64, (cuuint32_t)W, (cuuint32_t)(gemm::BK / W + 2), 1};
  const cuuint32_t estr[4] = {1, 1, 1, 1};
  return enc(map, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 4, const_cast<void*>(x), dims, strides, box, estr,
             CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
             CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}
template <int W>
static int launch_conv_wgrad_halo(const void* x, int N, int H, int Ci, const void* dz, float* c, int Co, int batch,
                                  int rpb, int64_t sc, cudaStream_t s) {
  CUtensorMap mdz, mx;
  if (!make_map_mn(&mdz, dz, Co, rpb, batch, (int64_t)rpb * Co) || !make_wg_halo_map(&mx, x, N, H, W, Ci))
    return ERR_CUDA;
  const int smem = gemm::WghSmem<W>::TOTAL + 1024;
  static bool attr = false;
  if (!attr) {
    if (cudaFuncSetAttribute(gemm::conv_wgrad_halo_kernel<W>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem) !=
        cudaSuccess)
      return ERR_CUDA;
    attr = true;
  }
  const int tiles = batch * 3 * (Ci / 64);
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  gemm::conv_wgrad_halo_kernel<W><<<tiles < sms ? tiles : sms, gemm::WGH_THREADS, smem, s>>>(mdz, mx, c, batch, rpb, H,
                                                                                            sc, Ci, Co);
  return cudaGetLastError() == cudaSuccess ? OK : ERR_CUDA;
}
template <int W, bool OUT_BF16>
static int launch_conv_halo(const void* x, int N, int H, const void* w, void* c, int Co, cudaStream_t s) {
  CUtensorMap mx, mw;
  if (!make_halo_map(&mx, x, N, H, W) || !make_map(&mw, w, Co, 9 * 64, 64, 1, (int64_t)Co * 9 * 64)) return ERR_CUDA;
  auto kern = gemm::conv_halo_kernel<W, OUT_BF16>;
  const int smem = gemm::HaloSmem<W>::TOTAL + 1024;
  static bool attr = false;
  if (!attr) {
    if (cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem) != cudaSuccess) return ERR_CUDA;
    attr = true;
  }
  const int M = N * H * W, tiles = (M + gemm::BM - 1) / gemm::BM;
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  kern<<<tiles < sms ? tiles : sms, gemm::HALO_THREADS, smem, s>>>(mx, mw, c, M, Co, H);
  return cudaGetLastError() == cudaSuccess ? OK : ERR_CUDA;
}

struct GemmShape {
  const void *a, *b;
  void* c;
  int M, N, K, batch;
  int64_t sa, sb, sc;  // batch strides of A, B and C in elements
  GemmEpi epi;
  bool mn;  // A, B MN-major: C[e] = A[e]^T B[e] with A[e] stored [K][M], B[e] stored [K][N]
  int aim = 0;  // implicit convolution operand (see AIM); x / geometry below
  gemm::ConvGeom cg{};
  int xN = 0, xH = 0, xW = 0, xC = 0;
};

template <int BN, int STAGES, bool OUT_BF16, bool MN, int AIM = 0>
static int launch_gemm(const GemmShape& g, int grid, cudaStream_t s) {
  const int M = g.M, N = g.N, K = g.K;
  CUtensorMap ma, mb, mc, mc2;
  bool in_ok;
  if (AIM == 1 || AIM == 3)
    in_ok = make_im2col_map(&ma, g.a, g.xN, g.xH, g.xW, g.xC, g.cg, gemm::BM) &&
            make_map(&mb, g.b, N, K, BN, g.batch, g.sb);
  else if (AIM == 2)
    in_ok = make_map_mn(&ma, g.a, M, K, g.batch, g.sa) && make_im2col_map(&mb, g.b, g.xN, g.xH, g.xW, g.xC, g.cg, 64);
  else if (AIM == 4)
    in_ok = make_map(&ma, g.a, M, K, gemm::BM, g.batch, g.sa) && make_map_mn(&mb, g.b, N, K, g.batch, g.sb);
  else
    in_ok = MN ? make_map_mn(&ma, g.a, M, K, g.batch, g.sa) && make_map_mn(&mb, g.b, N, K, g.batch, g.sb)
               : make_map(&ma, g.a, M, K, gemm::BM, g.batch, g.sa) && make_map(&mb, g.b, N, K, BN, g.batch, g.sb);
  if (!in_ok ||
      !make_store_map(&mc, g.c, M, N, g.batch, g.sc, OUT_BF16) ||
      !make_store_map(&mc2, g.epi.out2 ? (const void*)g.epi.out2 : g.c, M, N, g.batch, g.sc, OUT_BF16))
    return ERR_CUDA;
  auto kern = gemm::gemm_bf16_tn_kernel<BN, STAGES, OUT_BF16, MN, AIM>;
  const int smem = gemm::Smem<BN, STAGES, AIM == 3 ? gemm::RB_KB : 0>::TOTAL + 1024;
  static bool attr = false;
  if (!attr) {
    if (cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem) != cudaSuccess)
      return ERR_CUDA;
    attr = true;
  }
  const int tiles = ((M + gemm::BM - 1) / gemm::BM) * ((N + BN - 1) / BN) * g.batch;
  if (grid <= 0) {
    int dev = 0, sms = 148;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    grid = sms;
  }
  if (grid > tiles) grid = tiles;
  kern<<<grid, gemm::THREADS, smem, s>>>(ma, mb, mc, mc2, M, N, K, g.batch, g.epi, g.cg);
  return cudaGetLastError() == cudaSuccess ? OK : ERR_CUDA;
}

template <int STAGES, bool OUT_BF16, bool MN, int EW = gemm::EPI_WARPS, int AIM = 0, int NB = 2>
static int launch_gemm_pair(const GemmShape& g, int grid, cudaStream_t s) {
  const int M = g.M, N = g.N, K = g.K;
  CUtensorMap ma, mb, mc, mc2;
  const bool in_ok =
      AIM == 1   ? make_im2col_map(&ma, g.a, g.xN, g.xH, g.xW, g.xC, g.cg, gemm::BM) &&
                     make_map(&mb, g.b, N, K, gemm::PAIR_BN / 2, g.batch, g.sb)
      : AIM == 2 ? make_map_mn(&ma, g.a, M, K, g.batch, g.sa) &&
                     make_im2col_map(&mb, g.b, g.xN, g.xH, g.xW, g.xC, g.cg, 64)
      : AIM == 4 ? make_map(&ma, g.a, M, K, gemm::BM, g.batch, g.sa) && make_map_mn(&mb, g.b, N, K, g.batch, g.sb)
      : MN     ? make_map_mn(&ma, g.a, M, K, g.batch, g.sa) && make_map_mn(&mb, g.b, N, K, g.batch, g.sb)
               : make_map(&ma, g.a, M, K, gemm::BM, g.batch, g.sa) &&
                     make_map(&mb, g.b, N, K, gemm::PAIR_BN / 2, g.batch, g.sb);
  if (!in_ok ||
      !make_store_map(&mc, g.c, M, N, g.batch, g.sc, OUT_BF16) ||
      !make_store_map(&mc2, g.epi.out2 ? (const void*)g.epi.out2 : g.c, M, N, g.batch, g.sc, OUT_BF16))
    return ERR_CUDA;
  auto kern = gemm::gemm_bf16_tn_pair_kernel<STAGES, OUT_BF16, MN, EW, AIM, NB>;
  const int smem = gemm::PairSmem<STAGES, EW, NB>::TOTAL + 1024;
  static bool attr = false;
  if (!attr) {
    if (cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem) != cudaSuccess)
      return ERR_CUDA;
    attr = true;
  }
  const int tiles = (M / gemm::PAIR_M) * (N / gemm::PAIR_BN) * g.batch;
  if (grid <= 0) {
    int dev = 0, sms = 148;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    grid = sms;
  }
  grid &= ~1;  // CTA pairs
  if (grid < 2) grid = 2;
  if (grid > 2 * tiles) grid = 2 * tiles;
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(grid);
  cfg.blockDim = dim3(64 + 32 * EW);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = s;
  cudaLaunchAttribute attr_[1];
  attr_[0].id = cudaLaunchAttributeClusterDimension;
  attr_[0].val.clusterDim.x = 2;
  attr_[0].val.clusterDim.y = 1;
  attr_[0].val.clusterDim.z = 1;
  cfg.attrs = attr_;
  cfg.numAttrs = 1;
  return cudaLaunchKernelEx(&cfg, kern, ma, mb, mc, mc2, M, N, K, g.batch, g.epi, g.cg) == cudaSuccess ? OK : ERR_CUDA;
}

static int gemm_variant() {  // BT_GEMM_VARIANT=1 forces the 1-CTA kernel (tests, measurements)
  const char* e = getenv("BT_GEMM_VARIANT");
  return e ? atoi(e) : 0;
}

// 256 x 256 CTA-pair tiles when M and N allow it, else 128 x {256, 128, 64} tiles; ragged M / N / K
// edges are zero-filled by the TMA loads and clipped by the TMA stores (all deterministic)
template <bool MN, int AIM = 0>
static int launch_any(const GemmShape& g, int out_bf16, int grid, cudaStream_t s) {
  constexpr int SP = gemm::EPI_WARPS == 8 ? 5 : 3, S256 = gemm::EPI_WARPS == 8 ? 3 : 2,
                S64 = gemm::EPI_WARPS == 8 ? 6 : 4, S128 = gemm::EPI_WARPS == 8 ? 5 : 3;
  if (g.M % 256 == 0 && g.N % 256 == 0 && gemm_variant() != 1) {
    if (g.epi.kind == EPI_FFN_FWD || g.epi.kind == EPI_FFN_BWD) {  // ALU-heavy epilogues: 16 epilogue warps
      static const int ew = getenv("BT_FFN_EW") ? atoi(getenv("BT_FFN_EW")) : 16;  // A/B measurements
      if (ew == 8) return launch_gemm_pair<SP, true, MN, gemm::EPI_WARPS, AIM>(g, grid, s);
      if (ew == 81 && gemm::EPI_WARPS == 8) return launch_gemm_pair<6, true, MN, 8, AIM, 1>(g, grid, s);  // A/B
      // 16 warps x ONE staging box each (a box is re-staged only after its last store has read it; a chunk's
      // ALU work is far longer than that read) leaves room for 5 k-block stages instead of 3
      static const int nb = getenv("BT_FFN_NB") ? atoi(getenv("BT_FFN_NB")) : 1;  // A/B measurements
      if (nb == 2) return launch_gemm_pair<3, true, MN, 16, AIM>(g, grid, s);
      return launch_gemm_pair<5, true, MN, 16, AIM, 1>(g, grid, s);
    }
    // one staging box per epilogue warp makes room for a 6th k-block stage: 1-5% per GEMM at the C4 shapes
    // (tools/gemm_list.py); BT_PAIR_S6=0 restores 5 stages x 2 boxes (A/B)
    static const int s6 = getenv("BT_PAIR_S6") ? atoi(getenv("BT_PAIR_S6")) : 1;
    if (s6 && gemm::EPI_WARPS == 8)
      return out_bf16 ? launch_gemm_pair<6, true, MN, gemm::EPI_WARPS, AIM, 1>(g, grid, s)
                      : launch_gemm_pair<6, false, MN, gemm::EPI_WARPS, AIM, 1>(g, grid, s);
    return out_bf16 ? launch_gemm_pair<SP, true, MN, gemm::EPI_WARPS, AIM>(g, grid, s)
                    : launch_gemm_pair<SP, false, MN, gemm::EPI_WARPS, AIM>(g, grid, s);
  }
  if (g.N % 256 == 0)
    return out_bf16 ? launch_gemm<256, S256, true, MN, AIM>(g, grid, s)
                    : launch_gemm<256, S256, false, MN, AIM>(g, grid, s);
  if (g.N <= 64)  // narrow outputs (64-channel convolutions)
    return out_bf16 ? launch_gemm<64, S64, true, MN, AIM>(g, grid, s) : launch_gemm<64, S64, false, MN, AIM>(g, grid, s);
  return out_bf16 ? launch_gemm<128, S128, true, MN, AIM>(g, grid, s)
                  : launch_gemm<128, S128, false, MN, AIM>(g, grid, s);
}
// mn: 0 = A and B K-major (C = A.B^T); 1 = both MN-major (C = A^T.B); 2 = A K-major, B MN-major (C = A.B
// with B stored [K][N]) -- the same UMMAs over the same k order, so the same bits as mode 0 on B^T.
int gemm_bf16_launch_any(const void* a, const void* b, void* c, int batch, int M, int N, int K, int64_t sa,
                         int64_t sb, int64_t sc, int out_bf16, int grid, const GemmEpi& epi, int mn, cudaStream_t s) {
  const GemmShape g{a, b, c, M, N, K, batch, sa, sb, sc, epi, mn == 1};
  if (epi.kind == EPI_FFN_FWD || epi.kind == EPI_FFN_BWD) out_bf16 = 1;
  if (mn == 2) return launch_any<false, 4>(g, out_bf16, grid, s);
  return mn ? launch_any<true>(g, out_bf16, grid, s) : launch_any<false>(g, out_bf16, grid, s);
}
// Implicit-GEMM convolution products (1-CTA tiles).  fwd: C[Ho*Wo*N][Co] = im2col(x) . W^T with W [Co][K],
// K = taps * Ci.  wgrad: C[e][Co][K] = dz[e]^T im2col(x)[e], dz [rows][Co], rows_per_batch output pixels per
// batch entry (one EST), batch entries `batch`, C entries sc apart.
int gemm_conv_launch(int wgrad, const void* x, int xN, int xH, int xW, int Ci, int Ho, int Wo, int KH, int KW,
                     int stride, int pad, const void* other, void* c, int Co, int batch, int rows_per_batch,
                     int64_t sc, int out_bf16, cudaStream_t s) {
  GemmShape g{};
  g.cg = gemm::ConvGeom{Ho, Wo, stride, pad, KW, Ci / 64, rows_per_batch};
  g.xN = xN;
  g.xH = xH;
  g.xW = xW;
  g.xC = Ci;
  g.epi.kind = EPI_STORE;
  g.c = c;
  const int K = KH * KW * Ci;
  constexpr int S64 = gemm::EPI_WARPS == 8 ? 6 : 4, S128 = gemm::EPI_WARPS == 8 ? 5 : 3;
  if (!wgrad) {
    g.a = x;
    g.b = other;
    g.M = xN * Ho * Wo;
    g.N = Co;
    g.K = K;
    g.batch = 1;
    g.sb = (int64_t)Co * K;
    g.sc = (int64_t)g.M * Co;
    g.aim = 1;
    // 3x3 / stride 1 / pad 1, 64 input channels, Co <= 64, whole-row 128-pixel tiles: the halo form
    if (Ci == 64 && KH == 3 && KW == 3 && stride == 1 && pad == 1 && Ho == xH && Wo == xW && Co <= 64 &&
        (Co % 8) == 0 && (xW == 32 || xW == 16) && (xH * xW) % gemm::BM == 0 && getenv("BT_CONV_HALO0") == nullptr) {
      if (xW == 32)
        return out_bf16 ? launch_conv_halo<32, true>(x, xN, xH, other, c, Co, s)
                        : launch_conv_halo<32, false>(x, xN, xH, other, c, Co, s);
      return out_bf16 ? launch_conv_halo<16, true>(x, xN, xH, other, c, Co, s)
                      : launch_conv_halo<16, false>(x, xN, xH, other, c, Co, s);
    }
    constexpr int SRB = gemm::EPI_WARPS == 8 ? 5 : 7;  // A-only stages beside the 72 KB resident filter
    if (Co <= 64 && K <= 64 * gemm::RB_KB && getenv("BT_CONV_RB0") == nullptr)
      return out_bf16 ? launch_gemm<64, SRB, true, false, 3>(g, 0, s) : launch_gemm<64, SRB, false, false, 3>(g, 0, s);
    if (Co <= 64)
      return out_bf16 ? launch_gemm<64, S64, true, false, 1>(g, 0, s) : launch_gemm<64, S64, false, false, 1>(g, 0, s);
    if (Co % gemm::PAIR_BN == 0 && g.M % gemm::PAIR_M == 0 && getenv("BT_CONV_FWD_PAIR0") == nullptr) {
      constexpr int SP = gemm::EPI_WARPS == 8 ? 5 : 3;
      return out_bf16 ? launch_gemm_pair<SP, true, false, gemm::EPI_WARPS, 1>(g, 0, s)
                      : launch_gemm_pair<SP, false, false, gemm::EPI_WARPS, 1>(g, 0, s);
    }
    return out_bf16 ? launch_gemm<128, S128, true, false, 1>(g, 0, s) : launch_gemm<128, S128, false, false, 1>(g, 0, s);
  }
  g.a = other;  // dz [batch * rows_per_batch][Co]
  g.b = x;
  g.M = Co;
  g.N = K;
  g.K = rows_per_batch;
  g.batch = batch;
  g.sa = (int64_t)rows_per_batch * Co;
  g.sc = sc;
  g.mn = true;
  g.aim = 2;
  // 3x3 / stride 1 / pad 1, 64 or 128 channels in and out at W = 32 / 16 (layers 1 and 2): the halo form
  // (three taps per UMMA)
  if ((Ci == 64 || Ci == 128) && (Co == 64 || Co == 128) && KH == 3 && KW == 3 && stride == 1 && pad == 1 &&
      (xW == 32 || xW == 16) && Wo == xW && Ho == xH && rows_per_batch % gemm::BK == 0 && !out_bf16 &&
      getenv("BT_CONV_WG_HALO0") == nullptr)
    return xW == 32 ? launch_conv_wgrad_halo<32>(x, xN, xH, Ci, other, (float*)c, Co, batch, rows_per_batch, sc, s)
                    : launch_conv_wgrad_halo<16>(x, xN, xH, Ci, other, (float*)c, Co, batch, rows_per_batch, sc, s);
  // whole 256 x 256 CTA-pair tiles (Co, KH*KW*Ci multiples of 256): half the operand bytes per flop
  if (Co % gemm::PAIR_M == 0 && K % gemm::PAIR_BN == 0 && getenv("BT_CONV_WG_PAIR0") == nullptr) {
    constexpr int SP = gemm::EPI_WARPS == 8 ? 5 : 3;
    return out_bf16 ? launch_gemm_pair<SP, true, true, gemm::EPI_WARPS, 2>(g, 0, s)
                    : launch_gemm_pair<SP, false, true, gemm::EPI_WARPS, 2>(g, 0, s);
  }
  return out_bf16 ? launch_gemm<128, S128, true, true, 2>(g, 0, s) : launch_gemm<128, S128, false, true, 2>(g, 0, s);
}

int gemm_bf16_tn_launch_epi(const void* a, const void* b, void* c, int batch, int M, int N, int K, int64_t sa,
                            int64_t sb, int64_t sc, int out_bf16, int grid, const GemmEpi& epi, cudaStream_t s) {
  return gemm_bf16_launch_any(a, b, c, batch, M, N, K, sa, sb, sc, out_bf16, grid, epi, 0, s);
}
int gemm_bf16_tn_launch(const void* a, const void* b, void* c, int batch, int M, int N, int K, int64_t sa,
                        int64_t sb, int64_t sc, int out_bf16, int grid, cudaStream_t s) {
  GemmEpi epi{};
  epi.kind = EPI_STORE;
  return gemm_bf16_tn_launch_epi(a, b, c, batch, M, N, K, sa, sb, sc, out_bf16, grid, epi, s);
}

}  // namespace bt
