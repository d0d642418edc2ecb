/*
 * bittrain_b200.h -- C-ABI of the B200-native deterministic elastic
 * data-parallel step (the drop-in for the reference's run_minibatch path).
 *
 * The reference (`bittrain` 0.1.0, /root/reference/pkg/src/bittrain) is pure
 * Python with no FFI; its boundary is the Python API.  Each entry point below
 * replaces one reference function (cited file:line) and is what a ctypes /
 * cffi binding of that function would call.  The Python
 * package paper_2208_14228_b200 is exactly such a binding and keeps the
 * reference's names, argument meaning and exception classes.
 *
 * Conventions
 *  - Plain pointers and sizes only.  Pointers suffixed _dev (and all pointers
 *    inside bt_mlp_args / bt_reduce_args) are caller-owned DEVICE memory;
 *    nothing is allocated inside.  `stream` is a cudaStream_t (NULL = legacy).
 *  - Every call is stream-ordered and asynchronous except bt_step_status,
 *    the bt_host_* helpers and the IPC/peer helpers.
 *  - Return value: 0 = ok, else a status that maps 1:1 onto errors.py:
 *      1 InputError  2 ConfigError  3 StateError  4 ProgressError
 *      5 NumericError  6 CorruptionError  7 FormatError  8 VersionError
 *      9 CUDA/launch failure.  bt_last_error() returns this thread's message.
 *  - Device-detected errors (non-finite gradient, diverged replica) are
 *    written to a 4-word device status block `flags` {status, detail, step,
 *    spare}; the status word is sticky (later launches on the same block are
 *    no-ops) and is decoded by bt_step_status.
 */
#ifndef BITTRAIN_B200_H
#define BITTRAIN_B200_H

#include <stdint.h>

#include "../paper_2208_14228_b200/csrc/bt_mlp.cuh"
#include "../paper_2208_14228_b200/csrc/bt_reduce.cuh"

#ifdef __cplusplus
extern "C" {
#endif

#define BT_ABI_VERSION 1

int bt_abi_version(void);
const char *bt_last_error(void);
int bt_device_count(void);

/* ---------------- L0 numeric foundation: host-side sequential pieces ----
 * These are inherently serial (a Fisher-Yates chain, a byte-serial hash) and
 * run on the host in native code. */
uint64_t bt_host_mix64(uint64_t x);                                  /* prng.py:27-35 */
uint64_t bt_host_derive_stream(const uint64_t *words, int32_t n);    /* prng.py:59-69 */
uint64_t bt_host_fnv1a64(const void *data, int64_t nbytes);          /* prng.py:72-78 */
int bt_host_shuffled_range(int64_t n, uint64_t state, int32_t *out); /* prng.py:81-93 */
/* epoch_indices: out is [workers][steps_per_epoch*micro]             sampling.py:63-82 */
int bt_host_epoch_indices(uint64_t seed, uint64_t epoch, int64_t n, int32_t workers, int32_t micro,
                          int32_t shuffle, int32_t *out);
/* layout_arrival_perm: kind_fnv[e] = fnv1a64(utf-8 device kind)       buckets.py:70-82 */
int bt_host_layout_arrival_perm(int64_t nparams, int32_t nexec, const uint64_t *kind_fnv,
                                const int64_t *threads, int32_t *perm);
/* per-parameter ring-chunk rotation start pos*nrep//len(bucket)       buckets.py:119-122 */
int bt_host_rotation_table(int32_t nbuckets, const int32_t *sizes, const int32_t *idx, int32_t nrep,
                           int64_t nparams, int32_t *rot);

/* ---------------- L0 on device ------------------------------------------ */
/* n draws of a splitmix64 stream starting at draw `first` (counter form)   prng.py:38-56 */
int bt_splitmix64_draws(uint64_t state, uint64_t first, int64_t n, uint64_t *raw_dev, double *uniform_dev,
                        void *stream);
/* reduce_sum(values, Sequential|Tree(fanin)); fanin 0 = Sequential        reduction.py:51-62 */
int bt_reduce_sum_f64(const double *values_dev, int64_t n, int32_t fanin, double *out_dev, void *stream);

/* ---------------- L1 model ops --------------------------------------------- */
/* math.tanh as the reference's libm computes it (glibc tanh + FMA expm1)   model.py:148 */
int bt_tanh_f64(const double *x_dev, int64_t n, double *out_dev, void *stream);
/* ToyModel.init_random: (u*2-1)*scale per parameter                      model.py:58-66 */
int bt_init_random(uint64_t seed, double scale, int64_t n, double *out_dev, void *stream);
/* forward_backward for E ESTs at once (one CTA group per EST block).     model.py:107-196
 * rows_dev is the split_by_rank global batch [B*E_total][9] (row r of EST k at
 * r*E_total+k); est_fanin_dev [E]; rng/stat arrays are read and advanced in
 * place; losses_out [E]; grads_out [E][161].  rank_override >= 0 replaces the
 * TrackedStat rank of EST 0 (the single-worker seam). */
int bt_fwd_bwd_mlp_f64(const double *params_dev, const double *rows_dev, int32_t E, int32_t est_base,
                       int32_t E_total, int32_t B, const int32_t *est_fanin_dev, double rate,
                       int64_t rank_override, uint64_t *rng_io_dev, double *stat_mean_io_dev,
                       uint64_t *stat_count_io_dev, double *losses_out_dev, double *grads_out_dev,
                       int32_t *flags_dev, void *stream);
/* The whole mini-batch, K consecutive times, in ONE launch: data -> replica
 * check -> fwd/bwd of every EST -> fixed-order allreduce (executor 0's
 * variant, rank-keyed) -> /E -> momentum SGD -> mirror to every replica.
 *                                                           engine.py:271-329 */
int bt_mlp_step(const bt_mlp_args *args, void *stream);
/* bt_mlp_step, then the K x E_total per-EST losses and the 4-word status block copied into
 * caller-owned HOST buffers and the stream synchronised: the whole of one run_minibatch /
 * run_steps call in one entry point (losses_host may be NULL).  status_host may be NULL when the
 * device status block directly follows the K x E_total losses (args->flags == args->losses + K*E_total):
 * then ONE copy of the losses and the 4 status words lands in losses_host, the words at its tail.
 * In that layout, with losses_host pinned and the single-device compact build running, there is no copy
 * at all: the kernel's epilogue writes the losses and status words into losses_host (mapped) and then a
 * per-thread done word (system-scope release) that the call spins on -- the call returns when the
 * results are in host memory, without a stream synchronisation (the stream may still be retiring the
 * kernel: later work on it stays ordered).  BT_HOST_SIGNAL=0 restores copy + synchronise.
 *                                                                      engine.py:271-329 */
int bt_mlp_run(const bt_mlp_args *args, double *losses_host, int32_t *status_host, void *stream);
/* bt_mlp_run with the sampler's host work inside the call: the index lists of epochs [first_epoch,
 * first_epoch + n_epochs) are computed on the host (native Fisher-Yates seeded seed ^ epoch, dealt
 * round-robin: sampling.py:63-82) into stage_host (pinned, n_epochs * E_total * spe * B int32); the
 * launch reads them from stage_host through its mapped device address (zero-copy, once, in the prologue;
 * BT_LISTS_ZC=0: copied first) and they are copied to lists_dev on the stream after the launch, for
 * later calls of the same epochs (args->lists / epoch_base are taken from here).
 * Replaces the reference's per-step DataPipeline.batch + forward_backward + allreduce + sgd_step
 * (engine.py:271-329) for K mini-batches with host inputs and host outputs, one call. */
int bt_mlp_run_sampled(const bt_mlp_args *args, uint64_t seed, int64_t dataset_n, int32_t shuffle,
                       int64_t first_epoch, int32_t n_epochs, int32_t *stage_host, int32_t *lists_dev,
                       double *losses_host, int32_t *status_host, void *stream);
/* Blocks until no copy queued by bt_mlp_run_sampled still reads stage_host (call before re-filling it). */
int bt_stage_wait(const void *stage_host);
/* The multi-device form (bt_mlp_args.n_dev > 1): the n launches of one lock-step exchange group,
 * launch i on CUDA device devices[i] / streams[i]; all are queued before any host wait (they
 * exchange EST slots with each other every mini-batch), then each device's losses (its own EST
 * columns) and status words are copied to the host buffers and every stream synchronised.
 * The whole of one multi-GPU run_minibatch / run_steps call.             engine.py:271-329 */
int bt_mlp_run_group(const bt_mlp_args *const *args, const int32_t *devices, void *const *streams, int32_t n,
                     double *const *losses_host, int32_t *const *status_host);
/* Same launch with per-stage clock64 sums accumulated into timing_dev[0..4]
 * (rows+tanh, output chain, gradients, allreduce fold, update) and the step
 * count into timing_dev[5]; the compact build also adds its prologue, epilogue and whole-CTA
 * cycles into timing_dev[9..11] (profiling; thread 0 of CTA 0's view; 16 words). */
int bt_mlp_step_profiled(const bt_mlp_args *args, uint64_t *timing_dev, void *stream);
/* 1 when the fused (fuse_reduce = 1) step fits on chip for these args (E_total
 * slots in shared memory), else 0: use grads-only + bt_reduce_update. */
int bt_mlp_fused_fits(const bt_mlp_args *args);
/* Default ESTs-per-CTA for a shape (single CTA when the whole step fits). */
int bt_mlp_pick_est_per_cta(int32_t E, int32_t B);

/* ---------------- L2 communication: the deterministic reducer ------------ */
/* allreduce(replicas, bucket_map, variant) [+ sgd_step], one shard.
 *                                        buckets.py:85-124 + model.py:199-213 */
int bt_reduce_update(const bt_reduce_args *args, void *stream);
/* sgd_step, out of place; NumericError reported through flags.            model.py:199-213 */
int bt_sgd_step_f64(const double *params_dev, const double *vel_dev, const double *grads_dev, int64_t n,
                    double lr, double mu, double *params_out_dev, double *vel_out_dev, int32_t *flags_dev,
                    void *stream);

/* ---------------- deterministic tensor-core GEMM (C3/C4 model stack) ------
 * C[M][N] = A[M][K] * B[N][K]^T, bf16 inputs (K contiguous), fp32 accumulate
 * in TMEM, C fp32 (out_dtype 0) or bf16 (1).  tcgen05 + TMA, one CTA (pair)
 * per output tile, fixed K order: the bits depend only on the inputs and the
 * shape, never on `grid` (0 = one CTA per SM) or the GPU.  Ragged M / N / K
 * are zero-filled by the TMA loads and clipped by the TMA stores; rows must be
 * 16-byte aligned (K % 8 == 0, N % 8 == 0), pointers 16-byte aligned.
 *                                         analogue of model.py:141-192's dense products */
int bt_gemm_bf16_tn(const void *a_dev, const void *b_dev, void *c_dev, int32_t M, int32_t N, int32_t K,
                    int32_t out_dtype, int32_t grid, void *stream);
/* Batched form: C[e] = A[e] * B[e]^T for e < batch; A[e] at a_dev + e*stride_a elements, B[e] at
 * b_dev + e*stride_b, C[e] at c_dev + e*M*N (e.g. one weight gradient per EST, each its own GEMM,
 * reduced afterwards by bt_reduce_update in EST-rank order). */
int bt_gemm_bf16_tn_batched(const void *a_dev, const void *b_dev, void *c_dev, int32_t batch, int32_t M, int32_t N,
                            int32_t K, int64_t stride_a, int64_t stride_b, int32_t out_dtype, int32_t grid,
                            void *stream);

/* ---------------- per-EST transformer FFN step (C4 slice, no reference) ----
 * The kernels between the GEMMs of a BERT-style FFN sublayer trained by E ESTs
 * (tokens of local EST e are rows [e*Te, (e+1)*Te)); all randomness is keyed
 * by (seed, est_base + e, step, element) and all sums have a fixed shape.
 * Activations bf16, GEMM outputs fp32.                  analogue of model.py:141-196 */
int bt_ffn_data(uint64_t seed, int64_t step, int32_t est_base, int32_t E, int32_t Te, int32_t D, void *x_dev,
                float *target_dev, void *stream);
int bt_ffn_fwd_act(const float *h_dev, const float *b1_dev, uint64_t seed, int64_t step, int32_t est_base, int32_t E,
                   int32_t Te, int32_t F, float p, void *hpre_dev, void *d_dev, void *stream);
/* The FFN's GEMMs with the element ops fused into the epilogue (no fp32 round trip):
 * kind 1 (forward):  h = A*B^T + bias -> c = bf16(h), out2 = bf16(dropout(gelu(h)))
 * kind 2 (backward): c = bf16((A*B^T) * dropout_scale * gelu'(aux))   (aux = bf16 pre-activations)
 * rows are tokens, row r belongs to EST est_base + r / Te; same determinism as bt_gemm_bf16_tn.
 * kind | BT_GEMM_B_MN: B is stored [K][N] (C = A*B: the weights as stored, no transposed copy). */
#define BT_GEMM_B_MN 0x100
int bt_gemm_bf16_ffn(const void *a_dev, const void *b_dev, void *c_dev, int32_t M, int32_t N, int32_t K, int32_t kind,
                     const float *bias_dev, const void *aux_dev, void *out2_dev, uint64_t seed, int64_t step,
                     int32_t est_base, int32_t Te, float p, int32_t grid, void *stream);
/* bt_gemm_bf16_ffn with kind FFN_BWD and, when colpart_dev is set, the column sums of the bf16 output over
 * every 32-row block written to colpart_dev[M/32][N] (fp32; each block: even rows ascending + odd rows
 * ascending) -- the bias gradient's partials, without re-reading the output (fold: bt_colsum_fold). */
int bt_gemm_bf16_ffn_cs(const void *a_dev, const void *b_dev, void *c_dev, int32_t M, int32_t N, int32_t K,
                        int32_t kind, const float *bias_dev, const void *aux_dev, void *out2_dev, float *colpart_dev,
                        uint64_t seed, int64_t step, int32_t est_base, int32_t Te, float p, int32_t grid,
                        void *stream);
/* out[e*out_stride + c] = sum_k part[(e*chunks + k)*C + c], k ascending (per-leaf fold of column partials) */
int bt_colsum_fold(const float *part_dev, int32_t E, int32_t chunks, int32_t C, float *out_dev, int64_t out_stride,
                   void *stream);
/* partials_dev: E*64 floats of scratch; loss_dev[E] = sum 0.5*(y-target)^2 / Te; dy = (y-target)/Te */
int bt_ffn_out(const float *y_dev, const float *b2_dev, const float *target_dev, int32_t E, int32_t Te, int32_t D,
               void *dy_dev, float *partials_dev, float *loss_dev, void *stream);
int bt_ffn_bwd_act(const float *dd_dev, const void *hpre_dev, uint64_t seed, int64_t step, int32_t est_base,
                   int32_t E, int32_t Te, int32_t F, float p, void *dh_dev, void *stream);
/* out[e][c] = sum_r in[e][r][c] (bf16 in, fp32 out): ascending 64-row chunks summed ascending, then
 * the chunk sums in order (fixed association).  scratch_dev: E*ceil(R/64)*C floats, or NULL. */
int bt_colsum_bf16(const void *in_dev, int32_t E, int32_t R, int32_t C, float *out_dev, float *scratch_dev,
                   void *stream);
/* out[e][c][r] = bf16(in[e][r][c]); in is bf16 (in_f32 = 0) or fp32 (1) */
int bt_transpose_to_bf16(const void *in_dev, int32_t in_f32, int32_t E, int32_t R, int32_t C, void *out_dev,
                         void *stream);
int bt_cast_f32_bf16(const float *in_dev, int64_t n, void *out_dev, void *stream);
/* General form of the GEMM: batch strides for A, B and C (stride_c = 0: M*N) -- e.g. per-EST weight
 * gradients written straight into each EST's slot of a [E][P] gradient buffer; bias_dev (or NULL)
 * is added to every row in the epilogue (C = A*B^T + bias). */
int bt_gemm_bf16_tn_ex(const void *a_dev, const void *b_dev, void *c_dev, int32_t batch, int32_t M, int32_t N,
                       int32_t K, int64_t stride_a, int64_t stride_b, int64_t stride_c, int32_t out_dtype,
                       const float *bias_dev, int32_t grid, void *stream);
/* mn_major = 1: both operands MN-major, C[e] = A[e]^T * B[e] with A[e] stored [K][M] and B[e] stored
 * [K][N] (M / N contiguous) -- e.g. a per-EST weight gradient dW_e = dY_e^T X_e read straight from the
 * token-major activations dY [T][M], X [T][N] (stride_a = Te*M, stride_b = Te*N; no transposes).
 * mn_major = 2: A K-major [M][K], B MN-major stored [K][N]: C = A * B -- a dX product dY * W reading the
 * weight W [out][in] as stored (bit-identical to mode 0 on W^T: the same UMMAs in the same k order). */
int bt_gemm_bf16_ex(const void *a_dev, const void *b_dev, void *c_dev, int32_t batch, int32_t M, int32_t N, int32_t K,
                    int64_t stride_a, int64_t stride_b, int64_t stride_c, int32_t out_dtype, const float *bias_dev,
                    int32_t mn_major, int32_t grid, void *stream);
/* Implicit-GEMM convolution on the tcgen05 GEMM with TMA im2col-mode loads (no im2col matrix in HBM).
 * x: NHWC bf16 [xN][xH][xW][Ci], Ci % 64 == 0; filter KH x KW, stride, pad; output grid Ho x Wo.
 * wgrad = 0: c[xN*Ho*Wo][Co] = im2col(x) . W^T, other = W [Co][KH*KW*Ci] (K order (kh, kw, ci)).
 * wgrad = 1: c[e] (e < batch, stride_c apart) [Co][KH*KW*Ci] = dz[e]^T im2col(x)[e], other = dz
 *            [xN*Ho*Wo][Co]; each batch entry is rows_per_batch (% 64 == 0) output pixels (one EST).
 * Same tiles, same K order -- the same bits -- as the explicit im2col + bt_gemm_bf16_ex. */
int bt_gemm_conv(int32_t wgrad, const void *x_dev, int32_t xN, int32_t xH, int32_t xW, int32_t Ci, int32_t Ho,
                 int32_t Wo, int32_t KH, int32_t KW, int32_t stride, int32_t pad, const void *other_dev, void *c_dev,
                 int32_t Co, int32_t batch, int32_t rows_per_batch, int64_t stride_c, int32_t out_dtype, void *stream);
/* bt_colsum_bf16 with out[e][c] at out_dev + e*out_stride + c */
int bt_colsum_bf16_strided(const void *in_dev, int32_t E, int32_t R, int32_t C, float *out_dev, int64_t out_stride,
                           float *scratch_dev, void *stream);

/* C4 input / output layers (csrc/bt_embed.cu; synthetic token ids from splitmix64
 * mod the vocabulary).  Per sequence of 128 tokens: ids from the EST's token stream, `npred` masked
 * positions by a partial Fisher-Yates of the EST's mask stream (sorted), [MASK] = mask_id at those
 * inputs; mrow / mlabel: the masked rows of the launch and their original ids. */
int bt_bert_tokens(uint64_t seed, int64_t step, const int64_t *step_dev, int32_t est_base, int32_t E, int32_t seqs,
                   int32_t vocab, int32_t npred, int32_t mask_id, int32_t *ids_dev, int32_t *mrow_dev,
                   int32_t *mlabel_dev, void *stream);
/* x32[t] = wemb[ids[t]] + pemb[t % 128] (fp32), xb = bf16(x32) */
int bt_bert_embed_fwd(const int32_t *ids_dev, const float *wemb_dev, const float *pemb_dev, int32_t T, int32_t D,
                      float *x32_dev, void *xb_dev, void *stream);
/* bf16 row gather out[r] = in[rows[r]] / scatter dst[rows[r]] = src[r] (other rows of dst zeroed) */
int bt_rows_gather(const void *in_dev, const int32_t *rows_dev, int32_t R, int32_t D, void *out_dev, void *stream);
int bt_rows_scatter(const void *src_dev, const int32_t *rows_dev, int32_t R, int32_t npred, int32_t T, int32_t D,
                    void *dst_dev, void *stream);
/* Masked-LM cross-entropy: logits [R][vocab_pad] fp32 (columns >= vocab ignored); per-row loss, the
 * per-EST mean over its rows_per_est rows (row order), dlogits = (softmax - onehot) / rows_per_est
 * as bf16 [R][vocab_pad] (padding 0). */
int bt_bert_mlm_ce(const float *logits_dev, const int32_t *labels_dev, int32_t R, int32_t vocab, int32_t vocab_pad,
                   int32_t E, int32_t rows_per_est, void *dlogits_dev, float *row_loss_dev, float *loss_dev,
                   void *stream);
/* Embedding gradient without atomics: per gradient leaf, the (id, token) pairs sorted in shared
 * memory (a bitonic network); per distinct id the rows dx = dxa (bf16) + dxb (fp32) summed in token
 * order -- in chunks of 16 rows summed in parallel and folded in chunk order when an id repeats
 * ([MASK]) -- and ADDED to dwemb[leaf][id] (which holds the tied decoder's GEMM gradient);
 * dpemb[leaf][p] = the sum over the leaf's sequences, in order.  Scratch sizes from
 * bt_bert_embed_grad_scratch (int32 and fp32 element counts). */
int bt_bert_embed_grad_scratch(int32_t leaves, int32_t leaf_tokens, int32_t D, int64_t *ints_out,
                               int64_t *floats_out);
int bt_bert_embed_grad(const void *dxa_dev, const float *dxb_dev, const int32_t *ids_dev, int32_t leaves,
                       int32_t leaf_tokens, int32_t D, int32_t *scratch_dev, float *partial_dev, float *dwemb_dev,
                       float *dpemb_dev, int64_t leaf_stride, void *stream);
/* ---------------- per-EST BERT encoder step (C4, no reference) ------------
 * Post-LN BERT layer (attention with 64-wide heads over 128-token sequences,
 * LayerNorm, GELU FFN, hidden and attention-probability dropout).  Tokens of
 * local EST e are rows [e*Te, (e+1)*Te), Te % 128 == 0, D % 256 == 0.  Every
 * random draw is keyed by (seed, est_base + e, step, layer, element), every
 * sum has a shape fixed by the EST's own data: an EST's results do not depend
 * on which ESTs share the launch or the GPU.  step_dev (or NULL): read the step from device memory
 * instead of `step` (a CUDA graph of the whole step replays with an advancing counter).
 *                                                       analogue of model.py:107-196 */
int bt_bert_data(uint64_t seed, int64_t step, int32_t est_base, int32_t E, int32_t Te, int32_t D, float *x32_dev,
                 void *xb_dev, float *target_dev, const int64_t *step_dev, void *stream);
/* forward (backward = 0): ctx[T][D] = dropout(softmax(Q K^T / 8)) V per (sequence, head), qkv [T][3D] bf16;
 * backward (1): out = dqkv [T][3D] from qkv and dctx [T][D] (P recomputed bit-identically) */
int bt_bert_attn(int32_t backward, const void *qkv_dev, const void *dctx_dev, void *out_dev, int32_t E, int32_t Te,
                 int32_t D, int32_t heads, int32_t est_base, int32_t layers, int32_t layer, uint64_t seed, int64_t step,
                 float p, const int64_t *step_dev, void *stream);
/* bt_bert_attn with the softmax row statistics kept between the passes: the forward (tcgen05 path)
 * writes (-max * scale, 1 / sum) of every query row to stats_dev [E*Te/128 * heads][128] float2, the
 * backward reads them instead of recomputing (the same instruction sequence on the same S: the same
 * bits); stats_dev NULL: the backward recomputes them. */
int bt_bert_attn_ex(int32_t backward, const void *qkv_dev, const void *dctx_dev, void *out_dev, int32_t E,
                    int32_t Te, int32_t D, int32_t heads, int32_t est_base, int32_t layers, int32_t layer,
                    uint64_t seed, int64_t step, float p, const int64_t *step_dev, float *stats_dev, void *stream);
/* bt_bert_attn_ex with the attention-dropout keep bits: mbits_dev [E*Te/128*heads][128][4] uint32 (16-byte
 * aligned; row r of (sequence, head) item i at ((i*128 + r)*4), column c at bit c % 32 of word c / 32) --
 * written by the forward, read by the backward instead of drawing the masks again; NULL: draw them. */
int bt_bert_attn_ex2(int32_t backward, const void *qkv_dev, const void *dctx_dev, void *out_dev, int32_t E,
                     int32_t Te, int32_t D, int32_t heads, int32_t est_base, int32_t layers, int32_t layer, uint64_t seed,
                     int64_t step, float p, const int64_t *step_dev, float *stats_dev, uint32_t *mbits_dev,
                     void *stream);
/* x = resid + dropout(branch + bias); y = LayerNorm(x) * gamma + beta -> xsum (x), stats (mean, rstd)
 * [T][2], y32 (may be NULL), yb (bf16).  resid fp32 (the residual stream), branch bf16 (a GEMM output). */
int bt_bert_ln_fwd(const float *resid_dev, const void *branch_dev, const float *bias_dev, const float *gamma_dev,
                   const float *beta_dev, float *xsum_dev, float *stats_dev, float *y32_dev, void *yb_dev, int32_t E,
                   int32_t Te, int32_t D, int32_t est_base, int32_t layers, int32_t layer, int32_t site, uint64_t seed,
                   int64_t step, float p, float eps, const int64_t *step_dev, void *stream);
/* bt_bert_ln_fwd whose residual input is the previous LayerNorm's output recomputed from that LayerNorm's
 * input, (mean, rstd) and affine parameters -- the expression that produced its fp32 output, so the same
 * bits -- instead of a stored fp32 copy; y32_dev may be NULL (no fp32 output written) */
int bt_bert_ln_fwd_rc(const float *prev_xsum_dev, const float *prev_stats_dev, const float *prev_gamma_dev,
                      const float *prev_beta_dev, const void *branch_dev, const float *bias_dev, const float *gamma_dev,
                      const float *beta_dev, float *xsum_dev, float *stats_dev, float *y32_dev, void *yb_dev, int32_t E,
                      int32_t Te, int32_t D, int32_t est_base, int32_t layers, int32_t layer, int32_t site,
                      uint64_t seed, int64_t step, float p, float eps, const int64_t *step_dev, void *stream);
/* dx = LayerNorm'(dy1 + dy2) (dy1 bf16 from a GEMM, dy2 fp32 residual-path gradient or NULL),
 * dbranch = bf16(dropout'(dx)); part [E][Te/64][3][D] = per-64-row-chunk column sums of
 * (dy*xhat, dy, dropout'(dx)) */
int bt_bert_ln_bwd(const void *dy1_dev, const float *dy2_dev, const float *xsum_dev, const float *stats_dev,
                   const float *gamma_dev, float *dx_dev, void *dbranch_dev, float *part_dev, int32_t E, int32_t Te,
                   int32_t D, int32_t est_base, int32_t layers, int32_t layer, int32_t site, uint64_t seed,
                   int64_t step, float p, const int64_t *step_dev, void *stream);
/* chunk partials summed in chunk order -> dgamma/dbeta/dbias of EST e at + e*est_stride */
int bt_bert_ln_fold(const float *part_dev, int32_t E, int32_t Te, int32_t D, float *dgamma_dev, float *dbeta_dev,
                    float *dbias_dev, int64_t est_stride, void *stream);
/* loss[e] = sum 0.5*(y-target)^2 / Te, dy = bf16((y-target)/Te); partials_dev: E*64 floats */
int bt_bert_mse(const float *y_dev, const float *target_dev, int32_t E, int32_t Te, int32_t D, void *dy_dev,
                float *partials_dev, float *loss_dev, void *stream);
/* bf16 operand copies of fp32 master weights, one launch: wb[i] = bf16(w[i]) [rows][cols],
 * wt[i] = bf16(w[i])^T [cols][rows] */
int bt_cast_weights_bf16(const float *const *w_dev, void *const *wb_dev, void *const *wt_dev, const int32_t *rows,
                         const int32_t *cols, int32_t n, void *stream);

/* ---------------- per-EST ResNet-18 step with BatchNorm (C3, no reference) ----
 * NHWC bf16 activations; the images of local EST e are [e*B, (e+1)*B), its rows one
 * contiguous block.  Each EST normalises with its own micro-batch statistics and keeps
 * its own running statistics (slot [E] x run_stride); data are keyed by (seed, EST rank,
 * the EST's sampler cursor slot).  Convolutions are bt_gemm_bf16_ex products of
 * im2col matrices (forward, and the transposed convolution for dX as a gather).
 *                                                    analogue of model.py:94-104, 107-196 */
int bt_cnn_data(uint64_t seed, const int64_t *cursor_dev, int32_t est_base, int32_t E, int32_t B, void *x_dev,
                int32_t *labels_dev, void *stream);
/* col[(n,ho,wo)][(kh,kw,c)]: forward source (ho*s-p+kh, wo*s-p+kw); transposed = 1: source
 * ((ho+p-kh)/s, (wo+p-kw)/s) when exact (the dX gather of a stride-s convolution) */
int bt_cnn_im2col(const void *src_dev, void *col_dev, int32_t N, int32_t Hs, int32_t Ws, int32_t C, int32_t Ho,
                  int32_t Wo, int32_t KH, int32_t KW, int32_t stride, int32_t pad, int32_t transposed, void *stream);
/* per-EST column statistics over fixed 256-row chunks (1024 for mode 0 with C <= 64; C in {8, 16, 32, 64} or a multiple of 64), the
 * chunk partials folded in a fixed shape (32 lanes in chunk order, then a butterfly); mode 0 (one pass over z, shifted
 * by the EST's first row): mean, rstd and the running-statistics update of each EST's slot; mode 2:
 * backward sums (g, g*xhat) -> dbeta, dgamma of each EST's gradient slot (g = dy * [y > 0]).
 * part_dev: E * ceil(R/256) * 2 * C floats */
int bt_cnn_bn_stats(int32_t mode, const void *z_dev, const void *dy_dev, const void *y_dev, float *mean_dev,
                    float *rstd_dev, float *sg_dev, float *sgx_dev, float *part_dev, float *run_mean_dev,
                    float *run_var_dev, int64_t run_stride, float *dgamma_dev, float *dbeta_dev, int64_t grad_stride,
                    int32_t E, int32_t R, int32_t C, float eps, void *stream);
/* y = [relu](gamma (z - mean) rstd + beta [+ res]) */
int bt_cnn_bn_apply(const void *z_dev, const void *res_dev, const float *mean_dev, const float *rstd_dev,
                    const float *gamma_dev, const float *beta_dev, int32_t E, int32_t R, int32_t C, int32_t relu,
                    void *y_dev, void *stream);
/* dz = gamma rstd (g - S_g/R - xhat S_gx/R), g = dy [y > 0] */
int bt_cnn_bn_bwd(const void *z_dev, const void *dy_dev, const void *y_dev, const float *mean_dev,
                  const float *rstd_dev, const float *sg_dev, const float *sgx_dev, const float *gamma_dev, int32_t E,
                  int32_t R, int32_t C, void *dz_dev, void *stream);
/* out = a + (y ? b [y > 0] : b), n elements (bf16) */
int bt_cnn_add(const void *a_dev, const void *b_dev, const void *y_dev, int64_t n, void *out_dev, void *stream);
/* zero insertion: up [N][s*Hs][s*Ws][C] = src [N][Hs][Ws][C] at multiples of s, else 0 (bf16): the dX of a
 * stride-s convolution as a stride-1 convolution of `up` with the flipped filter */
int bt_cnn_upsample(const void *src_dev, int64_t N, int32_t Hs, int32_t Ws, int32_t C, int32_t s, void *up_dev,
                    void *stream);
/* stride-2 dX by output parity class (a, b): class filters out[i] [Ci][class_taps[i]][Co] (bf16) =
 * w[i] [Co][taps[i]][Ci] (fp32) at source taps tap_map[9*i + t], one launch for n <= 16 filters */
int bt_cnn_filter_taps(const float *const *w_dev, void *const *out_dev, const int32_t *co, const int32_t *taps,
                       const int32_t *ci, const int32_t *class_taps, const int32_t *tap_map, int32_t n, void *stream);
/* out [N][2Hs][2Ws][C] = a[2(y%2) + x%2][n][y/2][x/2] + b[...] (4 class pointers each, null = zero; bf16):
 * the parity classes of a stride-2 dX interleaved back, plus the shortcut's classes */
int bt_cnn_add_s2(const void *const *a_dev, const void *const *b_dev, void *out_dev, int64_t N, int32_t Hs, int32_t Ws,
                  int32_t C, void *stream);
/* avgpool 4x4 + fc 512->10 + softmax cross-entropy, forward and backward, one block per EST */
int bt_cnn_head(const void *x_dev, const int32_t *labels_dev, const float *w_dev, const float *b_dev, int32_t E,
                int32_t B, float *dw_dev, float *db_dev, int64_t grad_stride, float *loss_dev, void *dx_dev,
                void *stream);
/* out[e] (at out_dev + e*out_stride, n floats) = sum over sp ascending of part[e*splits + sp]: the fixed
 * split-K fold of per-EST weight gradients computed in pinned pixel splits */
int bt_fold_splits(const float *part_dev, int32_t E, int32_t splits, int64_t n, float *out_dev, int64_t out_stride,
                   void *stream);
/* master conv weights [Co][taps][Ci] fp32 -> wb [Co][taps*Ci] and wt [Ci][taps][Co] (bf16; taps reversed
 * where flip[i], for a stride-1 dX computed as a forward convolution of dz), one launch */
int bt_cnn_conv_weights(const float *const *w_dev, void *const *wb_dev, void *const *wt_dev, const int32_t *co,
                        const int32_t *taps, const int32_t *ci, const int32_t *flip, int32_t n, void *stream);

/* ---------------- L3 data ------------------------------------------------- */
/* make_dataset(seed, n, dim): [n][dim+1], x then y                       sampling.py:24-35 */
int bt_make_dataset(uint64_t seed, int64_t n, int32_t dim, double *out_dev, void *stream);
/* DataPipeline._produce for ESTs [est_base, est_base+E) at (epoch, local):
 * lists_dev is the epoch's [E_total][spe*B] lists; rows_out [E][B][9].  sampling.py:160-172 */
int bt_jitter_gather(const double *dataset_dev, const int32_t *lists_dev, int32_t E, int32_t est_base,
                     int32_t E_total, int32_t B, int64_t spe, uint64_t seed, int64_t epoch, int64_t local,
                     double jitter, double *rows_out_dev, void *stream);
/* forward_backward's dropout masks for `rows` rows of `units` units      model.py:151-161 */
int bt_dropout_mask(uint64_t state, int64_t rows, int32_t units, double rate, double *out_dev, void *stream);

/* ---------------- L4 runtime ---------------------------------------------- */
/* check_replica_agreement: R buffers of nbytes compared bytewise with buffer 0;
 * sets CorruptionError in flags.                                        engine.py:246-258 */
int bt_replica_check(const void *const *ptrs_dev, int32_t R, int64_t nbytes, int32_t *flags_dev, void *stream);
/* EST context/slot moves (elastic rescale), 128-bit vectorised, up to 64 pairs. */
int bt_est_slot_copy(void *const *dst_dev, const void *const *src_dev, const int64_t *bytes, int32_t count,
                     void *stream);
/* Parameter all-gather by peer stores: copy `n` elements of `dtype` from
 * src_dev to every dst in dst_dev[0..ndst) (bit copies, deterministic).   engine.py:313-315 */
int bt_allgather_params(int32_t dtype, const void *src_dev, void *const *dst_dev, int32_t ndst, int64_t n,
                        void *stream);
/* Stream-ordered copy between any two device (or peer / IPC-mapped / pinned host) addresses:
 * the guarded multi-rank reducer publishes each shard's status word with it. */
int bt_memcpy_async(void *dst, const void *src, int64_t nbytes, void *stream);
/* FNV-1a 64 of every `chunk`-byte slice of a device buffer (chunk % 16 == 0; the last slice may be
 * short) into out_dev [ceil(nbytes / chunk)]: the parallel half of the model-stack fingerprint
 * (runlog.device_fingerprint = host FNV-1a of these values).                   runlog.py:30-31 */
int bt_fnv1a64_chunks(const void *data_dev, int64_t nbytes, int64_t chunk, uint64_t *out_dev, void *stream);
/* Reset a status block to {0, INT32_MAX, 0, 0}. */
/* measurement helper: write `value` over bytes of buf_dev (16-byte aligned) -- the L2 flush between timed
 * launches, launched with the step kernels' shared-memory carveout preference */
int bt_l2_flush(void *buf_dev, int64_t bytes, uint32_t value, void *stream);
int bt_flags_reset(int32_t *flags_dev, void *stream);
/* Synchronise `stream`, read the status block; returns its status word. */
int bt_step_status(const int32_t *flags_dev, int32_t *detail_out, int32_t *step_out, void *stream);

/* ---------------- multi-GPU plumbing (one process per GPU) -------------- */
int bt_ipc_handle_size(void);
/* handle of the allocation containing dev_ptr, plus dev_ptr's byte offset in it */
int bt_ipc_get_handle(const void *dev_ptr, void *handle_out, int64_t *offset_out);
int bt_ipc_open_handle(const void *handle, void **dev_ptr_out);
int bt_ipc_close(void *dev_ptr);
int bt_enable_peer_access(int32_t peer_device);
/* stream-ordered signalling between GPUs: write a word when the stream gets
 * here (local or peer memory); make a stream wait until a word is >= value */
int bt_stream_write_u32(void *dev_ptr, uint32_t value, void *stream);
int bt_stream_wait_u32_geq(void *dev_ptr, uint32_t value, void *stream);

#ifdef __cplusplus
}
#endif

#endif /* BITTRAIN_B200_H */
