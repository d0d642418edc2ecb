// bt_embed.cu -- the input and output layers of the per-EST BERT step (C4: "synthetic
// token ids from splitmix64 mod 30522"): token / masked-LM data, the word + position embedding, the
// masked-LM cross-entropy over the vocabulary (decoder tied to the word embedding, as BERT does) and
// the embedding gradient.  The dense products around them (logits = y_m W^T + b, dy_m = dlogits W,
// dW_dec = dlogits^T y_m) are the deterministic tcgen05 GEMMs of bt_gemm.cu.
//
// EasyScale contract, as everywhere in the model stack: every draw is keyed by (seed, global EST rank,
// step, position) in counter form, and every reduction has a shape fixed by the EST's own data.  The
// embedding gradient is the classic nondeterminism site (a scatter-add: atomics in mainstream stacks);
// here it has NO atomics: each gradient leaf sorts its (token id, position) pairs in shared memory,
// and one warp per distinct id sums that id's rows in position order, after the decoder GEMM's
// contribution, into the leaf's slot -- the same bits whatever the launch grouping or GPU.
//
// Layout (launch of n ESTs, Te = S * 128 tokens each, leaves of g ESTs):
//   ids    [T] int32      input ids after masking ([MASK] at the masked positions)
//   mrow   [n*S*NP] int32  masked rows (token index within the launch), per sequence ascending
//   mlabel [n*S*NP] int32  the original id at each masked row (the MLM target)
//   logits [R][Vp] fp32, dlogits [R][Vp] bf16 (R = n*S*NP; columns >= V are padding, never a class)
#include <cuda_bf16.h>
#include <cuda_runtime.h>
#include <stdint.h>

#include "bt_common.cuh"

namespace bt {
namespace emb {

constexpr uint64_t TAG_TOK = 0x4245'5254'544f'4b4eull;   // "BERTTOKN" token ids
constexpr uint64_t TAG_MASK = 0x4245'5254'4d41'534bull;  // "BERTMASK" masked positions
constexpr int SEQ = 128;
constexpr int MAX_NP = 32;  // masked positions per sequence

__device__ __forceinline__ int64_t cur_step_e(int64_t step, const int64_t* step_dev) {
  return step_dev ? *step_dev : step;
}

// One CTA per sequence: thread t draws position t's id (raw % V of the EST's token stream at counter
// step*Te + t); thread 0 picks NP distinct positions by a partial Fisher-Yates over 0..127 (the
// mask stream at counters ((step*S + s)*NP + k)), sorts them, records them with their original ids,
// and replaces those input ids by mask_id.
__global__ void __launch_bounds__(SEQ) tokens_kernel(uint64_t seed, int64_t step_h, const int64_t* step_dev,
                                                     int est_base, int S, int V, int np, int mask_id, int32_t* ids,
                                                     int32_t* mrow, int32_t* mlabel) {
  const int64_t step = cur_step_e(step_h, step_dev);
  const int seq = blockIdx.x, e = seq / S, sl = seq - e * S, t = threadIdx.x;
  const int Te = S * SEQ;
  const uint64_t st = derive3(TAG_TOK, seed, (uint64_t)(est_base + e));
  __shared__ int32_t s_id[SEQ];
  __shared__ int32_t s_pos[SEQ];
  const int32_t id = (int32_t)(draw_raw(st, (uint64_t)step * Te + (uint64_t)sl * SEQ + t) % (uint64_t)V);
  s_id[t] = id;
  s_pos[t] = t;
  __syncthreads();
  if (t == 0) {
    const uint64_t sm = derive3(TAG_MASK, seed, (uint64_t)(est_base + e));
    for (int k = 0; k < np; ++k) {  // partial Fisher-Yates: position k <- a uniform pick of the rest
      const uint64_t raw = draw_raw(sm, ((uint64_t)step * S + sl) * np + k);
      const int j = k + (int)(raw % (uint64_t)(SEQ - k));
      const int tmp = s_pos[k];
      s_pos[k] = s_pos[j];
      s_pos[j] = tmp;
    }
    for (int a = 1; a < np; ++a) {  // ascending positions (insertion sort of <= 32)
      const int v = s_pos[a];
      int b = a - 1;
      while (b >= 0 && s_pos[b] > v) {
        s_pos[b + 1] = s_pos[b];
        --b;
      }
      s_pos[b + 1] = v;
    }
    for (int k = 0; k < np; ++k) {
      const int p = s_pos[k];
      mrow[seq * np + k] = seq * SEQ + p;
      mlabel[seq * np + k] = s_id[p];
    }
  }
  __syncthreads();
  bool masked = false;
  for (int k = 0; k < np; ++k) masked |= s_pos[k] == t;
  ids[seq * SEQ + t] = masked ? mask_id : id;
}

// x32[t] = W[ids[t]] + Pe[t % 128] (fp32, the residual stream's start), xb = bf16(x32)
__global__ void __launch_bounds__(256) embed_fwd_kernel(const int32_t* __restrict__ ids, const float* __restrict__ W,
                                                        const float* __restrict__ Pe, int T, int D, float* x32,
                                                        __nv_bfloat16* xb) {
  const int t = blockIdx.x;
  if (t >= T) return;
  const float* w = W + (size_t)ids[t] * D;
  const float* p = Pe + (size_t)(t % SEQ) * D;
  for (int c = threadIdx.x * 4; c < D; c += 256 * 4) {
    const float4 a = *(const float4*)(w + c), b = *(const float4*)(p + c);
    const float4 x = make_float4(a.x + b.x, a.y + b.y, a.z + b.z, a.w + b.w);
    *(float4*)(x32 + (size_t)t * D + c) = x;
    __nv_bfloat162 lo = __floats2bfloat162_rn(x.x, x.y), hi = __floats2bfloat162_rn(x.z, x.w);
    *(__nv_bfloat162*)(xb + (size_t)t * D + c) = lo;
    *(__nv_bfloat162*)(xb + (size_t)t * D + c + 2) = hi;
  }
}

// out[r] = in[rows[r]] (bf16 rows, D % 8 == 0)
__global__ void __launch_bounds__(128) gather_rows_kernel(const __nv_bfloat16* __restrict__ in,
                                                          const int32_t* __restrict__ rows, int R, int D,
                                                          __nv_bfloat16* __restrict__ out) {
  const int r = blockIdx.x;
  if (r >= R) return;
  const uint4* src = (const uint4*)(in + (size_t)rows[r] * D);
  uint4* dst = (uint4*)(out + (size_t)r * D);
  for (int c = threadIdx.x; c < D / 8; c += 128) dst[c] = src[c];
}

// dst[rows[r]] = src[r]; every other row of dst zero (one CTA per destination row: no races)
__global__ void __launch_bounds__(128) scatter_rows_kernel(const __nv_bfloat16* __restrict__ src,
                                                           const int32_t* __restrict__ rows, int R, int np, int T,
                                                           int D, __nv_bfloat16* __restrict__ dst) {
  const int t = blockIdx.x;
  if (t >= T) return;
  const int seq = t / SEQ;
  int r = -1;
  for (int k = 0; k < np; ++k)
    if (rows[seq * np + k] == t) r = seq * np + k;
  uint4* d = (uint4*)(dst + (size_t)t * D);
  const uint4* s = r >= 0 ? (const uint4*)(src + (size_t)r * D) : nullptr;
  for (int c = threadIdx.x; c < D / 8; c += 128) d[c] = s ? s[c] : make_uint4(0, 0, 0, 0);
}

// Cross-entropy of one masked row over the V classes (columns >= V are padding).  One read of the row
// for the statistics: each thread keeps an online (max, exp-sum) over its 4-column groups in
// ascending order, the 256 pairs are combined by a fixed tree; then dlogits = (softmax - onehot) *
// inv_rows (the EST's loss is the mean over its masked rows), bf16, zero in the padding;
// loss = log(sum) + max - logit[label].  Vp % 4 == 0.
constexpr int CE_THREADS = 256;
__device__ __forceinline__ void ms_combine(float& m, float& s, float m2, float s2) {
  const float mn = fmaxf(m, m2);
  s = (m == -INFINITY ? 0.f : s * __expf(m - mn)) + (m2 == -INFINITY ? 0.f : s2 * __expf(m2 - mn));
  m = mn;
}
__global__ void __launch_bounds__(CE_THREADS) ce_kernel(const float* __restrict__ logits,
                                                        const int32_t* __restrict__ labels, int V, int Vp,
                                                        float inv_rows, __nv_bfloat16* __restrict__ dlogits,
                                                        float* __restrict__ row_loss) {
  __shared__ float sm_m[CE_THREADS], sm_s[CE_THREADS];
  const int r = blockIdx.x;
  const float* l = logits + (size_t)r * Vp;
  float m = -INFINITY, s = 0.f;
  for (int c = threadIdx.x * 4; c < V; c += CE_THREADS * 4) {
    const float4 v = *(const float4*)(l + c);
    const float x[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
    for (int q = 0; q < 4; ++q)
      if (c + q < V) ms_combine(m, s, x[q], 1.f);
  }
  sm_m[threadIdx.x] = m;
  sm_s[threadIdx.x] = s;
  __syncthreads();
  for (int w = CE_THREADS / 2; w > 0; w >>= 1) {
    if (threadIdx.x < w) {
      float mm = sm_m[threadIdx.x], ss = sm_s[threadIdx.x];
      ms_combine(mm, ss, sm_m[threadIdx.x + w], sm_s[threadIdx.x + w]);
      sm_m[threadIdx.x] = mm;
      sm_s[threadIdx.x] = ss;
    }
    __syncthreads();
  }
  m = sm_m[0];
  s = sm_s[0];
  const int lab = labels[r];
  const float inv_s = 1.f / s;
  __nv_bfloat16* d = dlogits + (size_t)r * Vp;
  for (int c = threadIdx.x * 4; c < Vp; c += CE_THREADS * 4) {
    const float4 v = *(const float4*)(l + c);
    const float x[4] = {v.x, v.y, v.z, v.w};
    float g[4];
#pragma unroll
    for (int q = 0; q < 4; ++q)
      g[q] = c + q < V ? (__expf(x[q] - m) * inv_s - (c + q == lab ? 1.f : 0.f)) * inv_rows : 0.f;
    *(__nv_bfloat162*)(d + c) = __floats2bfloat162_rn(g[0], g[1]);
    *(__nv_bfloat162*)(d + c + 2) = __floats2bfloat162_rn(g[2], g[3]);
  }
  if (threadIdx.x == 0) row_loss[r] = __logf(s) + m - l[lab];
}
// The same cross-entropy with the row held in registers: 1024 threads per row, NV float4s each, so the
// logits are read from HBM once (the two-pass form above reads every row twice).  Exact row max (a max
// is order-free), then the exp sum per thread in column order, the warps' sums by a fixed butterfly and
// the 32 warps in order -- deterministic; then dlogits from the registers.
constexpr int CE_RT = 1024;
template <int NV>
__global__ void __launch_bounds__(CE_RT) ce_reg_kernel(const float* __restrict__ logits,
                                                      const int32_t* __restrict__ labels, int V, int Vp,
                                                      float inv_rows, __nv_bfloat16* __restrict__ dlogits,
                                                      float* __restrict__ row_loss) {
  __shared__ float sm_w[CE_RT / 32];
  const int r = blockIdx.x, tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const float* l = logits + (size_t)r * Vp;
  float4 x[NV];
  float m = -INFINITY;
#pragma unroll
  for (int k = 0; k < NV; ++k) {
    const int c = (tid + k * CE_RT) * 4;
    x[k] = c < Vp ? __ldcs((const float4*)(l + c)) : make_float4(-INFINITY, -INFINITY, -INFINITY, -INFINITY);
    if (c + 0 >= V) x[k].x = -INFINITY;
    if (c + 1 >= V) x[k].y = -INFINITY;
    if (c + 2 >= V) x[k].z = -INFINITY;
    if (c + 3 >= V) x[k].w = -INFINITY;
    m = fmaxf(m, fmaxf(fmaxf(x[k].x, x[k].y), fmaxf(x[k].z, x[k].w)));
  }
#pragma unroll
  for (int o = 16; o; o >>= 1) m = fmaxf(m, __shfl_xor_sync(0xffffffffu, m, o));
  if (lane == 0) sm_w[warp] = m;
  __syncthreads();
  m = sm_w[0];
#pragma unroll
  for (int w = 1; w < CE_RT / 32; ++w) m = fmaxf(m, sm_w[w]);
  __syncthreads();
  float s = 0.f;
#pragma unroll
  for (int k = 0; k < NV; ++k) {  // exp(-inf - m) = 0 for the padding
    s += __expf(x[k].x - m);
    s += __expf(x[k].y - m);
    s += __expf(x[k].z - m);
    s += __expf(x[k].w - m);
  }
#pragma unroll
  for (int o = 16; o; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
  if (lane == 0) sm_w[warp] = s;
  __syncthreads();
  s = sm_w[0];
#pragma unroll
  for (int w = 1; w < CE_RT / 32; ++w) s += sm_w[w];
  const int lab = labels[r];
  const float inv_s = 1.f / s;
  __nv_bfloat16* d = dlogits + (size_t)r * Vp;
#pragma unroll
  for (int k = 0; k < NV; ++k) {
    const int c = (tid + k * CE_RT) * 4;
    if (c >= Vp) continue;
    const float xv[4] = {x[k].x, x[k].y, x[k].z, x[k].w};
    float g[4];
#pragma unroll
    for (int q = 0; q < 4; ++q)
      g[q] = c + q < V ? (__expf(xv[q] - m) * inv_s - (c + q == lab ? 1.f : 0.f)) * inv_rows : 0.f;
    uint2 u;
    *(__nv_bfloat162*)&u.x = __floats2bfloat162_rn(g[0], g[1]);
    *(__nv_bfloat162*)&u.y = __floats2bfloat162_rn(g[2], g[3]);
    *(uint2*)(d + c) = u;
  }
  if (tid == 0) row_loss[r] = __logf(s) + m - l[lab];
}
// loss[e] = (sum of the EST's row losses, in row order) / rows_per_est
__global__ void ce_fold_kernel(const float* __restrict__ row_loss, int E, int rows_per_est, float* __restrict__ loss) {
  const int e = blockIdx.x * blockDim.x + threadIdx.x;
  if (e >= E) return;
  float acc = row_loss[(size_t)e * rows_per_est];
  for (int k = 1; k < rows_per_est; ++k) acc += row_loss[(size_t)e * rows_per_est + k];
  loss[e] = acc / (float)rows_per_est;
}

// Embedding gradient, step 1 (one CTA of 1024 threads per gradient leaf): sort the leaf's (id, token)
// pairs by id, then token (a bitonic network over 64-bit keys in shared memory), then cut the sorted
// list into per-id segments and each segment into EG_CH-row chunks -- all with block-wide prefix sums,
// no serial pass.  Outputs per leaf: seg_tok (sorted token indices), seg_first (segment starts),
// seg_n; chunks = {cfirst [segment], clo, cseg, cpix [chunk]} (cpix: the chunk's partial slot, -1 when
// its segment is a single chunk), n_chunks.
constexpr int EG_CH = 16;  // rows per chunk: a long segment is summed as chunks in parallel, then in order
constexpr int SORT_THREADS = 1024;
__device__ int block_scan_inclusive(int* a, int n, int* warp_tot) {  // in place; returns the total
  const int per = (n + SORT_THREADS - 1) / SORT_THREADS, lo = threadIdx.x * per;
  int run = 0;
  for (int i = lo; i < lo + per && i < n; ++i) run += a[i];
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  int x = run;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const int y = __shfl_up_sync(0xffffffffu, x, o);
    if (lane >= o) x += y;
  }
  if (lane == 31) warp_tot[w] = x;
  __syncthreads();
  if (w == 0) {
    int t = warp_tot[lane];
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int y = __shfl_up_sync(0xffffffffu, t, o);
      if (lane >= o) t += y;
    }
    warp_tot[lane] = t;
  }
  __syncthreads();
  int acc = x - run + (w > 0 ? warp_tot[w - 1] : 0);  // exclusive prefix of this thread's range
  for (int i = lo; i < lo + per && i < n; ++i) {
    acc += a[i];
    a[i] = acc;
  }
  const int total = warp_tot[31];
  __syncthreads();
  return total;
}
__global__ void __launch_bounds__(SORT_THREADS) sort_segments_kernel(const int32_t* __restrict__ ids, int leaf_tokens,
                                                                     int pow2, int32_t* __restrict__ seg_tok,
                                                                     int32_t* __restrict__ seg_first,
                                                                     int32_t* __restrict__ seg_n,
                                                                     int32_t* __restrict__ chunks,
                                                                     int32_t* __restrict__ n_chunks) {
  extern __shared__ uint64_t keys[];  // [pow2] keys, then 4 int arrays of [pow2]
  __shared__ int warp_tot[32];
  int* sa = (int*)(keys + pow2);
  int* sb = sa + pow2;
  int* sfirst = sb + pow2;
  int* sc = sfirst + pow2;
  const int leaf = blockIdx.x, N = leaf_tokens;
  const int32_t* id = ids + (size_t)leaf * N;
  for (int i = threadIdx.x; i < pow2; i += blockDim.x)
    keys[i] = i < N ? ((uint64_t)(uint32_t)id[i] << 32) | (uint32_t)i : ~0ull;
  __syncthreads();
  for (int k = 2; k <= pow2; k <<= 1) {
    for (int j = k >> 1; j > 0; j >>= 1) {
      for (int i = threadIdx.x; i < pow2; i += blockDim.x) {
        const int ixj = i ^ j;
        if (ixj > i) {
          const uint64_t a = keys[i], b = keys[ixj];
          const bool up = (i & k) == 0;
          if ((a > b) == up) {
            keys[i] = b;
            keys[ixj] = a;
          }
        }
      }
      __syncthreads();
    }
  }
  int32_t* tok = seg_tok + (size_t)leaf * N;
  for (int i = threadIdx.x; i < N; i += blockDim.x) {
    tok[i] = (int32_t)(keys[i] & 0xffffffffu);
    sa[i] = (i == 0 || (keys[i] >> 32) != (keys[i - 1] >> 32)) ? 1 : 0;  // segment heads
  }
  __syncthreads();
  const int nseg = block_scan_inclusive(sa, N, warp_tot);  // sa[i] = heads in [0, i]
  for (int i = threadIdx.x; i < N; i += blockDim.x)
    if (i == 0 || sa[i] != sa[i - 1]) sfirst[sa[i] - 1] = i;
  __syncthreads();
  for (int k = threadIdx.x; k < nseg; k += blockDim.x) {  // chunks per segment; partial slots per segment
    const int len = (k + 1 < nseg ? sfirst[k + 1] : N) - sfirst[k], nch = (len + EG_CH - 1) / EG_CH;
    sb[k] = nch;
    sc[k] = nch > 1 ? nch : 0;
  }
  __syncthreads();
  const int nc = block_scan_inclusive(sb, nseg, warp_tot);  // sb[k] = chunks of segments 0..k
  block_scan_inclusive(sc, nseg, warp_tot);
  int32_t* first = seg_first + (size_t)leaf * N;
  int32_t* cfirst = chunks + (size_t)leaf * 4 * N;  // [segment] first chunk
  int32_t* clo = cfirst + N;                        // [chunk] first sorted row
  int32_t* cseg = clo + N;                          // [chunk] segment
  int32_t* cpix = cseg + N;                         // [chunk] partial slot or -1
  for (int k = threadIdx.x; k < nseg; k += blockDim.x) {
    const int c1 = sb[k], c0 = k > 0 ? sb[k - 1] : 0, p0 = k > 0 ? sc[k - 1] : 0;
    first[k] = sfirst[k];
    cfirst[k] = c0;
    for (int c = c0; c < c1; ++c) {
      clo[c] = sfirst[k] + (c - c0) * EG_CH;
      cseg[c] = k;
      cpix[c] = c1 - c0 > 1 ? p0 + (c - c0) : -1;
    }
  }
  if (threadIdx.x == 0) {
    seg_n[leaf] = nseg;
    n_chunks[leaf] = nc;
  }
}

// Embedding gradient, step 2: one warp per (chunk c, leaf): the sum, in token order, of the chunk's
// <= EG_CH rows dx[t] = dxa[t] (bf16) + dxb[t] (fp32) (loads batched 8 rows at a time); a segment of one
// chunk adds it to dW_leaf[id] (on top of the decoder GEMM's contribution: one addition, a fixed
// association), a longer segment ([MASK]: every masked position of the leaf) writes it to its partial
// slot for step 3.  Each lane owns 8-column groups (16-byte bf16 / 2 x 16-byte fp32 loads).
constexpr int EG_WARPS = 8;
__device__ __forceinline__ void row8(const __nv_bfloat16* dxa, const float* dxb, size_t t, int D, int c, float* v) {
  const uint4 ra = *(const uint4*)(dxa + t * D + c);
  const float4 b0 = *(const float4*)(dxb + t * D + c), b1 = *(const float4*)(dxb + t * D + c + 4);
  const __nv_bfloat162* a2 = (const __nv_bfloat162*)&ra;
#pragma unroll
  for (int q = 0; q < 4; ++q) {
    const float2 f = __bfloat1622float2(a2[q]);
    v[2 * q] = f.x;
    v[2 * q + 1] = f.y;
  }
  v[0] += b0.x; v[1] += b0.y; v[2] += b0.z; v[3] += b0.w;
  v[4] += b1.x; v[5] += b1.y; v[6] += b1.z; v[7] += b1.w;
}
__device__ __forceinline__ void add8(float* w, const float* acc) {
  float4* wp = (float4*)w;
  float4 o0 = wp[0], o1 = wp[1];
  o0.x += acc[0]; o0.y += acc[1]; o0.z += acc[2]; o0.w += acc[3];
  o1.x += acc[4]; o1.y += acc[5]; o1.z += acc[6]; o1.w += acc[7];
  wp[0] = o0;
  wp[1] = o1;
}
__global__ void __launch_bounds__(32 * EG_WARPS) embed_chunk_kernel(
    const __nv_bfloat16* __restrict__ dxa, const float* __restrict__ dxb, const int32_t* __restrict__ ids,
    const int32_t* __restrict__ seg_tok, const int32_t* __restrict__ seg_first, const int32_t* __restrict__ seg_n,
    const int32_t* __restrict__ chunks, const int32_t* __restrict__ n_chunks, int leaf_tokens, int D,
    float* __restrict__ dW, int64_t leaf_stride, float* __restrict__ partial, int pslots) {
  const int leaf = blockIdx.y, lane = threadIdx.x & 31;
  const int c = blockIdx.x * EG_WARPS + (threadIdx.x >> 5);
  if (c >= n_chunks[leaf]) return;
  const int32_t* cfirst = chunks + (size_t)leaf * 4 * leaf_tokens;
  const int32_t *clo = cfirst + leaf_tokens, *cseg = clo + leaf_tokens, *cpix = cseg + leaf_tokens;
  const int32_t* tok = seg_tok + (size_t)leaf * leaf_tokens;
  const int32_t* first = seg_first + (size_t)leaf * leaf_tokens;
  const int k = cseg[c], ns = seg_n[leaf];
  const int seg_hi = k + 1 < ns ? first[k + 1] : leaf_tokens;
  const int lo = clo[c], hi = lo + EG_CH < seg_hi ? lo + EG_CH : seg_hi;
  const size_t t0 = (size_t)leaf * leaf_tokens;
  const int pix = cpix[c];
  float* out = pix < 0 ? dW + (size_t)leaf * leaf_stride + (size_t)ids[t0 + tok[lo]] * D
                       : partial + ((size_t)leaf * pslots + pix) * D;
  constexpr int U = 8;
  for (int col = lane * 8; col < D; col += 32 * 8) {
    float acc[8];
    for (int i0 = lo; i0 < hi; i0 += U) {
      float v[U][8];
#pragma unroll
      for (int j = 0; j < U; ++j) row8(dxa, dxb, t0 + tok[i0 + j < hi ? i0 + j : lo], D, col, v[j]);
#pragma unroll
      for (int j = 0; j < U; ++j)
        if (i0 + j < hi)
#pragma unroll
          for (int q = 0; q < 8; ++q) acc[q] = i0 + j == lo ? v[j][q] : acc[q] + v[j][q];
    }
    if (pix < 0) {
      add8(out + col, acc);
    } else {
      *(float4*)(out + col) = make_float4(acc[0], acc[1], acc[2], acc[3]);
      *(float4*)(out + col + 4) = make_float4(acc[4], acc[5], acc[6], acc[7]);
    }
  }
}
// Embedding gradient, step 3: one warp per multi-chunk segment: its chunk partials summed in chunk order,
// then added to dW_leaf[id] (one addition).
__global__ void __launch_bounds__(32 * EG_WARPS) embed_fold_kernel(
    const int32_t* __restrict__ ids, const int32_t* __restrict__ seg_tok, const int32_t* __restrict__ seg_first,
    const int32_t* __restrict__ seg_n, const int32_t* __restrict__ chunks, const int32_t* __restrict__ n_chunks,
    int leaf_tokens, int D, float* __restrict__ dW, int64_t leaf_stride, const float* __restrict__ partial,
    int pslots) {
  const int leaf = blockIdx.y, lane = threadIdx.x & 31;
  const int k = blockIdx.x * EG_WARPS + (threadIdx.x >> 5);
  const int ns = seg_n[leaf];
  if (k >= ns) return;
  const int32_t* cfirst = chunks + (size_t)leaf * 4 * leaf_tokens;
  const int32_t* cpix = cfirst + 3 * leaf_tokens;
  const int c0 = cfirst[k], c1 = k + 1 < ns ? cfirst[k + 1] : n_chunks[leaf];
  if (c1 - c0 < 2) return;
  const int32_t* tok = seg_tok + (size_t)leaf * leaf_tokens;
  const int32_t* first = seg_first + (size_t)leaf * leaf_tokens;
  float* w = dW + (size_t)leaf * leaf_stride + (size_t)ids[(size_t)leaf * leaf_tokens + tok[first[k]]] * D;
  const float* pbase = partial + (size_t)leaf * pslots * D;
  for (int col = lane * 8; col < D; col += 32 * 8) {
    float acc[8];
    for (int c = c0; c < c1; ++c) {
      const float* p = pbase + (size_t)cpix[c] * D + col;
      const float4 a = *(const float4*)p, b = *(const float4*)(p + 4);
      const float v[8] = {a.x, a.y, a.z, a.w, b.x, b.y, b.z, b.w};
#pragma unroll
      for (int q = 0; q < 8; ++q) acc[q] = c == c0 ? v[q] : acc[q] + v[q];
    }
    add8(w + col, acc);
  }
}

// Position-embedding gradient: dPe_leaf[p] = sum over the leaf's sequences, in order, of dx[seq*128+p]
__global__ void __launch_bounds__(256) pos_grad_kernel(const __nv_bfloat16* __restrict__ dxa,
                                                       const float* __restrict__ dxb, int seqs_per_leaf, int D,
                                                       float* __restrict__ dP, int64_t leaf_stride) {
  const int p = blockIdx.x, leaf = blockIdx.y;
  for (int c = threadIdx.x; c < D; c += 256) {
    float acc = 0.f;
    for (int s = 0; s < seqs_per_leaf; ++s) {
      const size_t t = ((size_t)leaf * seqs_per_leaf + s) * SEQ + p;
      const float v = __bfloat162float(dxa[t * D + c]) + dxb[t * D + c];
      acc = s == 0 ? v : acc + v;
    }
    dP[(size_t)leaf * leaf_stride + (size_t)p * D + c] = acc;
  }
}

}  // namespace emb

static int ok_or_cuda_e() { return cudaGetLastError() == cudaSuccess ? OK : ERR_CUDA; }

int emb_tokens_launch(uint64_t seed, int64_t step, const int64_t* step_dev, int est_base, int E, int S, int V, int np,
                      int mask_id, int32_t* ids, int32_t* mrow, int32_t* mlabel, cudaStream_t s) {
  if (np < 1 || np > emb::MAX_NP || V < 2 || S < 1 || E < 1) return ERR_INPUT;
  emb::tokens_kernel<<<E * S, emb::SEQ, 0, s>>>(seed, step, step_dev, est_base, S, V, np, mask_id, ids, mrow, mlabel);
  return ok_or_cuda_e();
}

int emb_fwd_launch(const int32_t* ids, const float* W, const float* Pe, int T, int D, float* x32, void* xb,
                   cudaStream_t s) {
  if (D % 4) return ERR_INPUT;
  emb::embed_fwd_kernel<<<T, 256, 0, s>>>(ids, W, Pe, T, D, x32, (__nv_bfloat16*)xb);
  return ok_or_cuda_e();
}

int emb_gather_launch(const void* in, const int32_t* rows, int R, int D, void* out, cudaStream_t s) {
  if (D % 8) return ERR_INPUT;
  emb::gather_rows_kernel<<<R, 128, 0, s>>>((const __nv_bfloat16*)in, rows, R, D, (__nv_bfloat16*)out);
  return ok_or_cuda_e();
}

int emb_scatter_launch(const void* src, const int32_t* rows, int R, int np, int T, int D, void* dst, cudaStream_t s) {
  if (D % 8) return ERR_INPUT;
  emb::scatter_rows_kernel<<<T, 128, 0, s>>>((const __nv_bfloat16*)src, rows, R, np, T, D, (__nv_bfloat16*)dst);
  return ok_or_cuda_e();
}

int emb_ce_launch(const float* logits, const int32_t* labels, int R, int V, int Vp, int E, int rows_per_est,
                  void* dlogits, float* row_loss, float* loss, cudaStream_t s) {
  if (R != E * rows_per_est || V > Vp || Vp % 4) return ERR_INPUT;
  const int nv = (Vp / 4 + emb::CE_RT - 1) / emb::CE_RT;  // float4s per thread of the register form
  const float ir = 1.f / (float)rows_per_est;
  __nv_bfloat16* dl = (__nv_bfloat16*)dlogits;
  if (nv <= 1) emb::ce_reg_kernel<1><<<R, emb::CE_RT, 0, s>>>(logits, labels, V, Vp, ir, dl, row_loss);
  else if (nv <= 2) emb::ce_reg_kernel<2><<<R, emb::CE_RT, 0, s>>>(logits, labels, V, Vp, ir, dl, row_loss);
  else if (nv <= 4) emb::ce_reg_kernel<4><<<R, emb::CE_RT, 0, s>>>(logits, labels, V, Vp, ir, dl, row_loss);
  else if (nv <= 8) emb::ce_reg_kernel<8><<<R, emb::CE_RT, 0, s>>>(logits, labels, V, Vp, ir, dl, row_loss);
  else emb::ce_kernel<<<R, emb::CE_THREADS, 0, s>>>(logits, labels, V, Vp, ir, dl, row_loss);
  emb::ce_fold_kernel<<<(E + 127) / 128, 128, 0, s>>>(row_loss, E, rows_per_est, loss);
  return ok_or_cuda_e();
}

// int32 scratch: seg_tok, seg_first, chunks (4 arrays) per leaf = 6 * leaf_tokens, + seg_n, n_chunks;
// fp32 partials: pslots rows of D per leaf (chunks of multi-chunk segments, <= 2 * leaf_tokens / EG_CH + 1)
int emb_grad_scratch(int leaves, int leaf_tokens, int D, int64_t* ints, int64_t* floats) {
  *ints = (int64_t)leaves * 6 * leaf_tokens + 2 * (int64_t)leaves;
  *floats = (int64_t)leaves * (2 * leaf_tokens / emb::EG_CH + 1) * D;
  return OK;
}
int emb_grad_launch(const void* dxa, const float* dxb, const int32_t* ids, int leaves, int leaf_tokens, int D,
                    int32_t* scratch, float* partial, float* dW, float* dP, int64_t leaf_stride, cudaStream_t s) {
  if (leaf_tokens % emb::SEQ) return ERR_INPUT;
  int pow2 = 1;
  while (pow2 < leaf_tokens) pow2 <<= 1;
  const size_t smem = (sizeof(uint64_t) + 4 * sizeof(int)) * (size_t)pow2;  // keys + 4 int arrays
  if (smem > 200 * 1024) return ERR_INPUT;
  static size_t attr = 0;
  if (smem > 48 * 1024 && smem > attr) {
    if (cudaFuncSetAttribute(emb::sort_segments_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024) !=
        cudaSuccess)
      return ERR_CUDA;
    attr = 200 * 1024;
  }
  const size_t T = (size_t)leaves * leaf_tokens;
  int32_t* seg_tok = scratch;
  int32_t* seg_first = seg_tok + T;
  int32_t* chunks = seg_first + T;
  int32_t* seg_n = chunks + 4 * T;
  int32_t* n_chunks = seg_n + leaves;
  const int pslots = 2 * leaf_tokens / emb::EG_CH + 1;
  emb::sort_segments_kernel<<<leaves, emb::SORT_THREADS, smem, s>>>(ids, leaf_tokens, pow2, seg_tok, seg_first,
                                                                     seg_n, chunks, n_chunks);
  const dim3 grid((leaf_tokens + emb::EG_WARPS - 1) / emb::EG_WARPS, leaves);
  emb::embed_chunk_kernel<<<grid, 32 * emb::EG_WARPS, 0, s>>>((const __nv_bfloat16*)dxa, dxb, ids, seg_tok, seg_first,
                                                              seg_n, chunks, n_chunks, leaf_tokens, D, dW, leaf_stride,
                                                              partial, pslots);
  emb::embed_fold_kernel<<<grid, 32 * emb::EG_WARPS, 0, s>>>(ids, seg_tok, seg_first, seg_n, chunks, n_chunks,
                                                             leaf_tokens, D, dW, leaf_stride, partial, pslots);
  emb::pos_grad_kernel<<<dim3(emb::SEQ, leaves), 256, 0, s>>>((const __nv_bfloat16*)dxa, dxb,
                                                              leaf_tokens / emb::SEQ, D, dP, leaf_stride);
  return ok_or_cuda_e();
}

}  // namespace bt
