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
// and one CTA per distinct id sums that id's rows in position order, after the decoder GEMM's
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

// Cross-entropy of one masked row over the V classes (columns >= V are padding): row max, then the
// exp-sum in a fixed order (each thread its strided columns ascending, a fixed tree across threads);
// loss = log(sum) + max - logit[label]; dlogits = (softmax - onehot) * inv_rows (the EST's loss is the
// mean over its masked rows), bf16, zero in the padding.
constexpr int CE_THREADS = 256;
__device__ __forceinline__ float block_reduce(float v, float* sm, bool is_max) {
  sm[threadIdx.x] = v;
  __syncthreads();
  for (int w = CE_THREADS / 2; w > 0; w >>= 1) {
    if (threadIdx.x < w) sm[threadIdx.x] = is_max ? fmaxf(sm[threadIdx.x], sm[threadIdx.x + w])
                                                  : sm[threadIdx.x] + sm[threadIdx.x + w];
    __syncthreads();
  }
  const float out = sm[0];
  __syncthreads();
  return out;
}
__global__ void __launch_bounds__(CE_THREADS) ce_kernel(const float* __restrict__ logits,
                                                        const int32_t* __restrict__ labels, int V, int Vp,
                                                        float inv_rows, __nv_bfloat16* __restrict__ dlogits,
                                                        float* __restrict__ row_loss) {
  __shared__ float sm[CE_THREADS];
  const int r = blockIdx.x;
  const float* l = logits + (size_t)r * Vp;
  float m = -INFINITY;
  for (int c = threadIdx.x; c < V; c += CE_THREADS) m = fmaxf(m, l[c]);
  m = block_reduce(m, sm, true);
  float s = 0.f;
  for (int c = threadIdx.x; c < V; c += CE_THREADS) s += __expf(l[c] - m);
  s = block_reduce(s, sm, false);
  const int lab = labels[r];
  const float inv_s = 1.f / s;
  __nv_bfloat16* d = dlogits + (size_t)r * Vp;
  for (int c = threadIdx.x; c < Vp; c += CE_THREADS) {
    const float g = c < V ? (__expf(l[c] - m) * inv_s - (c == lab ? 1.f : 0.f)) * inv_rows : 0.f;
    d[c] = __float2bfloat16_rn(g);
  }
  if (threadIdx.x == 0) row_loss[r] = __logf(s) + m - l[lab];
}
// loss[e] = (sum of the EST's row losses, in row order) / rows_per_est
__global__ void ce_fold_kernel(const float* __restrict__ row_loss, int E, int rows_per_est, float* __restrict__ loss) {
  const int e = blockIdx.x * blockDim.x + threadIdx.x;
  if (e >= E) return;
  float acc = row_loss[(size_t)e * rows_per_est];
  for (int k = 1; k < rows_per_est; ++k) acc += row_loss[(size_t)e * rows_per_est + k];
  loss[e] = acc / (float)rows_per_est;
}

// Embedding gradient, step 1 (one CTA per gradient leaf): sort the leaf's (id, token) pairs by id,
// then token (a bitonic sort of 64-bit keys in shared memory: a fixed network), and cut the sorted
// list into per-id segments: seg_tok[leaf][i] = sorted token indices, seg_first[leaf][k] = start of
// segment k, seg_n[leaf] = number of segments.
__global__ void __launch_bounds__(1024) sort_segments_kernel(const int32_t* __restrict__ ids, int leaf_tokens,
                                                             int pow2, int32_t* __restrict__ seg_tok,
                                                             int32_t* __restrict__ seg_first,
                                                             int32_t* __restrict__ seg_n) {
  extern __shared__ uint64_t keys[];
  const int leaf = blockIdx.x;
  const int32_t* id = ids + (size_t)leaf * leaf_tokens;
  for (int i = threadIdx.x; i < pow2; i += blockDim.x)
    keys[i] = i < leaf_tokens ? ((uint64_t)(uint32_t)id[i] << 32) | (uint32_t)i : ~0ull;
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
  int32_t* tok = seg_tok + (size_t)leaf * leaf_tokens;
  int32_t* first = seg_first + (size_t)leaf * leaf_tokens;
  for (int i = threadIdx.x; i < leaf_tokens; i += blockDim.x) tok[i] = (int32_t)(keys[i] & 0xffffffffu);
  __syncthreads();
  if (threadIdx.x == 0) {  // segment starts (sequential: a few thousand compares)
    int n = 0;
    for (int i = 0; i < leaf_tokens; ++i)
      if (i == 0 || (keys[i] >> 32) != (keys[i - 1] >> 32)) first[n++] = i;
    seg_n[leaf] = n;
  }
}

// Embedding gradient, step 2: CTA (segment k, leaf): dW_leaf[id] += sum over the segment's tokens, in
// token order, of dx[t] = dxa[t] (bf16) + dxb[t] (fp32) -- added to the decoder GEMM's contribution
// already in the slot (one addition of the segment sum: a fixed association).
__global__ void __launch_bounds__(256) embed_grad_kernel(const __nv_bfloat16* __restrict__ dxa,
                                                         const float* __restrict__ dxb, const int32_t* __restrict__ ids,
                                                         const int32_t* __restrict__ seg_tok,
                                                         const int32_t* __restrict__ seg_first,
                                                         const int32_t* __restrict__ seg_n, int leaf_tokens, int D,
                                                         float* __restrict__ dW, int64_t leaf_stride) {
  const int leaf = blockIdx.y, k = blockIdx.x;
  if (k >= seg_n[leaf]) return;
  const int32_t* tok = seg_tok + (size_t)leaf * leaf_tokens;
  const int32_t* first = seg_first + (size_t)leaf * leaf_tokens;
  const int lo = first[k], hi = k + 1 < seg_n[leaf] ? first[k + 1] : leaf_tokens;
  const size_t t0 = (size_t)leaf * leaf_tokens;
  const int id = ids[t0 + tok[lo]];
  float* w = dW + (size_t)leaf * leaf_stride + (size_t)id * D;
  for (int c = threadIdx.x; c < D; c += 256) {
    float acc = 0.f;
    for (int i = lo; i < hi; ++i) {
      const size_t t = t0 + tok[i];
      const float v = __bfloat162float(dxa[t * D + c]) + dxb[t * D + c];
      acc = i == lo ? v : acc + v;
    }
    w[c] += acc;
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
  if (R != E * rows_per_est || V > Vp) return ERR_INPUT;
  emb::ce_kernel<<<R, emb::CE_THREADS, 0, s>>>(logits, labels, V, Vp, 1.f / (float)rows_per_est,
                                               (__nv_bfloat16*)dlogits, row_loss);
  emb::ce_fold_kernel<<<(E + 127) / 128, 128, 0, s>>>(row_loss, E, rows_per_est, loss);
  return ok_or_cuda_e();
}

int emb_grad_launch(const void* dxa, const float* dxb, const int32_t* ids, int leaves, int leaf_tokens, int D,
                    int32_t* seg_tok, int32_t* seg_first, int32_t* seg_n, float* dW, float* dP, int64_t leaf_stride,
                    cudaStream_t s) {
  if (leaf_tokens % emb::SEQ) return ERR_INPUT;
  int pow2 = 1;
  while (pow2 < leaf_tokens) pow2 <<= 1;
  const size_t smem = sizeof(uint64_t) * (size_t)pow2;
  if (smem > 200 * 1024) return ERR_INPUT;
  static size_t attr = 0;
  if (smem > 48 * 1024 && smem > attr) {
    if (cudaFuncSetAttribute(emb::sort_segments_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024) !=
        cudaSuccess)
      return ERR_CUDA;
    attr = 200 * 1024;
  }
  emb::sort_segments_kernel<<<leaves, 1024, smem, s>>>(ids, leaf_tokens, pow2, seg_tok, seg_first, seg_n);
  emb::embed_grad_kernel<<<dim3(leaf_tokens, leaves), 256, 0, s>>>((const __nv_bfloat16*)dxa, dxb, ids, seg_tok,
                                                                   seg_first, seg_n, leaf_tokens, D, dW, leaf_stride);
  emb::pos_grad_kernel<<<dim3(emb::SEQ, leaves), 256, 0, s>>>((const __nv_bfloat16*)dxa, dxb,
                                                              leaf_tokens / emb::SEQ, D, dP, leaf_stride);
  return ok_or_cuda_e();
}

}  // namespace bt
