// bt_capi.cu -- extern "C" entry points (include/bittrain_b200.h).
// Validation + status mapping onto errors.py + launches.  No torch types.
#include <cuda_runtime.h>

#include <stdarg.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

#include <vector>

#include "../../include/bittrain_b200.h"
#include "bt_common.cuh"
#include "bt_ffn.cuh"

namespace bt {
struct MlpHostSignal {
  double* out;
  uint32_t* done;
  uint32_t seq;
};
int mlp_launch(const bt_mlp_args& a, cudaStream_t s, unsigned long long* timing = nullptr,
               const MlpHostSignal* hs = nullptr, bool* signaled = nullptr);
size_t mlp_smem_bytes(int nrows);
bool mlp_fused_fits(const bt_mlp_args& a);
bool mlp_xdev_supported(const bt_mlp_args& a);
int reduce_launch(const bt_reduce_args& a, cudaStream_t s);
int reduce_sum_launch(const double* v, int64_t n, int fanin, double* out, cudaStream_t s);
int sgd_launch(const double* p, const double* v, const double* g, int64_t n, double lr, double mu, double* po,
               double* vo, int32_t* flags, cudaStream_t s);
int make_dataset_launch(uint64_t seed, int64_t n, int dim, double* out, cudaStream_t s);
int init_random_launch(uint64_t seed, double scale, int64_t n, double* out, cudaStream_t s);
int draws_launch(uint64_t state, uint64_t first, int64_t n, uint64_t* raw, double* uni, cudaStream_t s);
int jitter_gather_launch(const double* dataset, const int32_t* lists, int E, int est_base, int E_total, int B,
                         int64_t spe, uint64_t seed, int64_t epoch, int64_t local, double jitter, double* rows_out,
                         cudaStream_t s);
int dropout_mask_launch(uint64_t state, int64_t rows, int units, double rate, double* out, cudaStream_t s);
int replica_check_launch(const void* const* ptrs, int R, int64_t nbytes, int32_t* flags, cudaStream_t s);
int slot_copy_launch(void* const* dst, const void* const* src, const int64_t* bytes, int count, cudaStream_t s);
int flags_reset_launch(int32_t* flags, cudaStream_t s);
int l2_flush_launch(void* buf, int64_t bytes, uint32_t v, cudaStream_t s);
int tanh_launch(const double* x, int64_t n, double* out, cudaStream_t s);
int gemm_bf16_tn_launch(const void* a, const void* b, void* c, int batch, int M, int N, int K, int64_t sa,
                        int64_t sb, int64_t sc, int out_bf16, int grid, cudaStream_t s);
int gemm_bf16_tn_launch_epi(const void* a, const void* b, void* c, int batch, int M, int N, int K, int64_t sa,
                            int64_t sb, int64_t sc, int out_bf16, int grid, const GemmEpi& epi, cudaStream_t s);
int gemm_conv_launch(int wgrad, const void* x, int xN, int xH, int xW, int Ci, int Ho, int Wo, int KH, int KW,
                     int stride, int pad, const void* other, void* c, int Co, int batch, int rows_per_batch,
                     int64_t sc, int out_bf16, cudaStream_t s);
int gemm_bf16_launch_any(const void* a, const void* b, void* c, int batch, int M, int N, int K, int64_t sa,
                         int64_t sb, int64_t sc, int out_bf16, int grid, const GemmEpi& epi, int mn, cudaStream_t s);
int ffn_data_launch(uint64_t seed, int64_t step, int est_base, int E, int Te, int D, void* X, float* target,
                    cudaStream_t s);
int ffn_fwd_act_launch(const float* H, const float* b1, uint64_t seed, int64_t step, int est_base, int E, int Te,
                       int F, float p, void* Hpre, void* Dout, cudaStream_t s);
int ffn_out_launch(const float* Y, const float* b2, const float* target, int E, int Te, int D, void* dY, float* part,
                   float* loss, cudaStream_t s);
int ffn_bwd_act_launch(const float* dD, const void* Hpre, uint64_t seed, int64_t step, int est_base, int E, int Te,
                       int F, float p, void* dH, cudaStream_t s);
int colsum_bf16_launch(const void* in, int E, int R, int C, float* out, float* scratch, cudaStream_t s);
int transpose_launch(const void* in, int in_f32, int E, int R, int C, void* out, cudaStream_t s);
int cast_f32_bf16_launch(const float* in, int64_t n, void* out, cudaStream_t s);
int colsum_fold_launch(const float* part, int E, int chunks, int C, float* out, int64_t ostride, cudaStream_t s);
int colsum_bf16_strided_launch(const void* in, int E, int R, int C, float* out, int64_t ostride, float* scratch,
                               cudaStream_t s);
int bert_attn_launch(int backward, const void* qkv, const void* dctx, void* out, int n_seq, int Dm, int H,
                     int seqs_per_est, int est_base, int L, int layer, uint64_t seed, int64_t step, float p,
                     const int64_t* step_dev, cudaStream_t s, float* stats, uint32_t* mbits);
int bert_ln_launch(int backward, const float* in1, const void* in2, const float* bias, const float* gamma,
                   const float* beta, float* xsum, float* stats, float* y32, void* yb, float* part, int E, int Te,
                   int D, int est_base, int L, int layer, int site, uint64_t seed, int64_t step, float p, float eps,
                   const int64_t* step_dev, cudaStream_t s, const float* rx = nullptr,
                   const float* rst = nullptr, const float* rg = nullptr, const float* rb = nullptr);
int bert_ln_fold_launch(const float* part, int E, int Te, int D, float* dg, float* db, float* dr, int64_t est_stride,
                        cudaStream_t s);
int bert_data_launch(uint64_t seed, int64_t step, int est_base, int E, int Te, int D, float* X32, void* Xb,
                     float* target, const int64_t* step_dev, cudaStream_t s);
int bert_mse_launch(const float* y, const float* tgt, int E, int Te, int D, void* dy, float* part, float* loss,
                    cudaStream_t s);
int bert_cast_weights_launch(const float* const* w, void* const* wb, void* const* wt, const int* R, const int* C, int n,
                             cudaStream_t s);
int cnn_data_launch(uint64_t seed, const int64_t* cursor, int est_base, int E, int B, void* x, int32_t* labels,
                    cudaStream_t s);
int cnn_fold_splits_launch(const float* part, int E, int splits, int64_t n, float* out, int64_t out_stride,
                           cudaStream_t s);
int cnn_im2col_launch(const void* src, void* col, int N, int Hs, int Ws, int C, int Ho, int Wo, int KH, int KW,
                      int stride, int pad, int transposed, cudaStream_t s);
int cnn_bn_stats_launch(int mode, const void* z, const void* dy, const void* y, float* mean, float* rstd,
                        float* sg, float* sgx, float* part, float* run_mean, float* run_var, int64_t run_stride,
                        float* dgamma, float* dbeta, int64_t grad_stride, int E, int R, int C, float eps,
                        cudaStream_t s);
int cnn_bn_apply_launch(const void* z, const void* res, const float* mean, const float* rstd, const float* gamma,
                        const float* beta, int E, int R, int C, int relu, void* y, cudaStream_t s);
int cnn_bn_bwd_launch(const void* z, const void* dy, const void* y, const float* mean, const float* rstd,
                      const float* sg, const float* sgx, const float* gamma, int E, int R, int C, void* dz,
                      cudaStream_t s);
int cnn_add_launch(const void* a, const void* b, const void* y, int64_t n, void* out, cudaStream_t s);
int cnn_upsample_launch(const void* src, int64_t N, int Hs, int Ws, int C, int s, void* up, cudaStream_t st);
int cnn_filter_taps_launch(const float* const* w, void* const* out, const int* Co, const int* T, const int* Ci,
                           const int* Tc, const int* src, int n, cudaStream_t s);
int cnn_add_s2_launch(const void* const* a, const void* const* b, void* out, int64_t N, int Hs, int Ws, int C,
                      cudaStream_t s);
int cnn_head_launch(const void* x, const int32_t* labels, const float* W, const float* bias, int E, int B, float* dW,
                    float* db, int64_t grad_stride, float* loss, void* dx, cudaStream_t s);
int cnn_conv_weights_launch(const float* const* w, void* const* wb, void* const* wt, const int* Co, const int* T,
                            const int* Ci, const int* flip, int n, cudaStream_t s);
int fnv_chunks_launch(const void* data, int64_t nbytes, int64_t chunk, uint64_t* out, cudaStream_t s);
int emb_tokens_launch(uint64_t seed, int64_t step, const int64_t* step_dev, int est_base, int E, int S, int V, int np,
                      int mask_id, int32_t* ids, int32_t* mrow, int32_t* mlabel, cudaStream_t s);
int emb_fwd_launch(const int32_t* ids, const float* W, const float* Pe, int T, int D, float* x32, void* xb,
                   cudaStream_t s);
int emb_gather_launch(const void* in, const int32_t* rows, int R, int D, void* out, cudaStream_t s);
int emb_scatter_launch(const void* src, const int32_t* rows, int R, int np, int T, int D, void* dst, cudaStream_t s);
int emb_ce_launch(const float* logits, const int32_t* labels, int R, int V, int Vp, int E, int rows_per_est,
                  void* dlogits, float* row_loss, float* loss, cudaStream_t s);
int emb_grad_scratch(int leaves, int leaf_tokens, int D, int64_t* ints, int64_t* floats);
int emb_grad_launch(const void* dxa, const float* dxb, const int32_t* ids, int leaves, int leaf_tokens, int D,
                    int32_t* scratch, float* partial, float* dW, float* dP, int64_t leaf_stride, cudaStream_t s);
}  // namespace bt

static thread_local char g_err[512];

static int fail(int code, const char* fmt, ...) __attribute__((format(printf, 2, 3)));
static int fail(int code, const char* fmt, ...) {
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(g_err, sizeof g_err, fmt, ap);
  va_end(ap);
  return code;
}
static int cuda_fail(const char* what) {
  cudaError_t e = cudaGetLastError();
  return fail(bt::ERR_CUDA, "%s: %s", what, cudaGetErrorString(e));
}
static int done(int st, const char* what) {
  if (st == bt::OK) {
    g_err[0] = 0;
    return 0;
  }
  if (st == bt::ERR_CUDA) return cuda_fail(what);
  return st;
}
#define STREAM(s) ((cudaStream_t)(s))

extern "C" {

int bt_abi_version(void) { return BT_ABI_VERSION; }
const char* bt_last_error(void) { return g_err; }
int bt_device_count(void) {
  int n = 0;
  if (cudaGetDeviceCount(&n) != cudaSuccess) {
    cudaGetLastError();
    return 0;
  }
  return n;
}

// ------------------------------------------------------------- host helpers
uint64_t bt_host_mix64(uint64_t x) { return bt::mix64(x); }

uint64_t bt_host_derive_stream(const uint64_t* words, int32_t n) {
  uint64_t s = bt::DERIVE_SEED;
  for (int i = 0; i < n; ++i) s = bt::mix64(s ^ words[i]);
  return s;
}

uint64_t bt_host_fnv1a64(const void* data, int64_t nbytes) {
  const unsigned char* p = (const unsigned char*)data;
  uint64_t h = 0xCBF29CE484222325ull;
  for (int64_t i = 0; i < nbytes; ++i) {
    h ^= p[i];
    h *= 0x100000001B3ull;
  }
  return h;
}

int bt_host_shuffled_range(int64_t n, uint64_t state, int32_t* out) {
  if (n < 0 || n > 0x7fffffff) return fail(bt::ERR_INPUT, "shuffled_range: bad n %lld", (long long)n);
  for (int64_t i = 0; i < n; ++i) out[i] = (int32_t)i;
  for (int64_t t = n - 1; t > 0; --t) {
    state += bt::GOLDEN_GAMMA;
    const uint64_t raw = bt::mix64(state);
    const int64_t k = (int64_t)(raw % (uint64_t)(t + 1));
    const int32_t tmp = out[t];
    out[t] = out[k];
    out[k] = tmp;
  }
  return 0;
}

int bt_host_epoch_indices(uint64_t seed, uint64_t epoch, int64_t n, int32_t workers, int32_t micro, int32_t shuffle,
                          int32_t* out) {
  if (workers < 1) return fail(bt::ERR_CONFIG, "total_workers must be >= 1");
  if (n < workers) return fail(bt::ERR_CONFIG, "dataset smaller than the worker count");
  if (micro < 1) return fail(bt::ERR_CONFIG, "micro_batch must be >= 1");
  const int64_t spe = n / ((int64_t)workers * micro);
  if (spe < 1) return fail(bt::ERR_CONFIG, "dataset smaller than one global batch");
  static thread_local std::vector<int32_t> order;  // (reused: an allocation per epoch shows on the e2e path)
  order.resize((size_t)n);
  if (shuffle) bt_host_shuffled_range(n, seed ^ epoch, order.data());
  else for (int64_t i = 0; i < n; ++i) order[(size_t)i] = (int32_t)i;
  const int64_t per = spe * micro;
  for (int32_t k = 0; k < workers; ++k)
    for (int64_t t = 0; t < per; ++t) out[(size_t)k * per + t] = order[(size_t)(t * workers + k)];
  return 0;
}

int bt_host_layout_arrival_perm(int64_t nparams, int32_t nexec, const uint64_t* kind_fnv, const int64_t* threads,
                                int32_t* perm) {
  std::vector<uint64_t> w;
  w.push_back(bt::TAG_BUCKET_ARRIVAL);
  w.push_back((uint64_t)nexec);
  for (int e = 0; e < nexec; ++e) {
    w.push_back(kind_fnv[e]);
    w.push_back((uint64_t)threads[e]);
  }
  return bt_host_shuffled_range(nparams, bt_host_derive_stream(w.data(), (int32_t)w.size()), perm);
}

int bt_host_rotation_table(int32_t nbuckets, const int32_t* sizes, const int32_t* idx, int32_t nrep, int64_t nparams,
                           int32_t* rot) {
  int64_t base = 0;
  for (int b = 0; b < nbuckets; ++b) {
    const int64_t blen = sizes[b];
    for (int64_t pos = 0; pos < blen; ++pos) {
      const int64_t p = idx[base + pos];
      if (p < 0 || p >= nparams) return fail(bt::ERR_INPUT, "bucket index %lld out of range", (long long)p);
      rot[p] = (int32_t)((pos * nrep) / blen);
    }
    base += blen;
  }
  if (base != nparams) return fail(bt::ERR_INPUT, "bucket map covers %lld parameters, expected %lld",
                                   (long long)base, (long long)nparams);
  return 0;
}

// ------------------------------------------------------------- device: L0
int bt_splitmix64_draws(uint64_t state, uint64_t first, int64_t n, uint64_t* raw_dev, double* uniform_dev,
                        void* stream) {
  if (n < 0) return fail(bt::ERR_INPUT, "negative draw count");
  if (n == 0) return 0;
  return done(bt::draws_launch(state, first, n, raw_dev, uniform_dev, STREAM(stream)), "bt_splitmix64_draws");
}

int bt_reduce_sum_f64(const double* values_dev, int64_t n, int32_t fanin, double* out_dev, void* stream) {
  if (fanin < 0) return fail(bt::ERR_CONFIG, "fanin must be positive, got %d", fanin);
  if (fanin == 1) return fail(bt::ERR_CONFIG, "Tree(1) never terminates in the reference; rejected");
  if (n < 0) return fail(bt::ERR_INPUT, "negative length");
  return done(bt::reduce_sum_launch(values_dev, n, fanin, out_dev, STREAM(stream)), "bt_reduce_sum_f64");
}

// ------------------------------------------------------------- device: L1
int bt_tanh_f64(const double* x_dev, int64_t n, double* out_dev, void* stream) {
  if (n < 0) return fail(bt::ERR_INPUT, "negative length");
  if (n == 0) return 0;
  return done(bt::tanh_launch(x_dev, n, out_dev, STREAM(stream)), "bt_tanh_f64");
}

int bt_init_random(uint64_t seed, double scale, int64_t n, double* out_dev, void* stream) {
  return done(bt::init_random_launch(seed, scale, n, out_dev, STREAM(stream)), "bt_init_random");
}

int bt_mlp_pick_est_per_cta(int32_t E, int32_t B) {
  if (E < 1 || B < 1) return 1;
  // Spread the ESTs over up to 8 CTAs of one thread-block cluster (one SM
  // each): a mini-batch is a latency-bound fp64 chain, so fewer rows per SM
  // means less issue contention; the clustered CTAs exchange gradient slots
  // through DSMEM with one cluster barrier per step.  Each CTA holds at most
  // 256 rows (shared-memory tile); beyond 8 CTAs the grid-barrier path is used.
  int epc = (E + 7) / 8;
  if ((int64_t)epc * B > 256) epc = 256 / B > 0 ? 256 / B : 1;
  return epc;
}

static int validate_mlp(const bt_mlp_args* a) {
  if (!a) return fail(bt::ERR_INPUT, "null args");
  if (a->E < 1 || a->E_total < 1 || a->est_base < 0 || a->est_base + a->E > a->E_total)
    return fail(bt::ERR_INPUT, "bad EST range [%d, %d) of %d", a->est_base, a->est_base + a->E, a->E_total);
  if (a->B < 1 || a->B > 256) return fail(bt::ERR_INPUT, "micro-batch %d outside [1, 256]", a->B);
  if (a->K < 1) return fail(bt::ERR_INPUT, "K must be >= 1");
  if (a->X < 1) return fail(bt::ERR_INPUT, "need at least one replica");
  if (a->est_per_cta < 1 || (int64_t)a->est_per_cta * a->B > 256)
    return fail(bt::ERR_INPUT, "est_per_cta*B must be in [1, 256]");
  if (a->n_dev < 0 || a->n_dev > BT_MAX_XDEV) return fail(bt::ERR_INPUT, "n_dev %d outside [0, %d]", a->n_dev, BT_MAX_XDEV);
  if (a->n_dev > 1) {
    if (a->dev_index < 0 || a->dev_index >= a->n_dev) return fail(bt::ERR_INPUT, "dev_index %d of %d", a->dev_index, a->n_dev);
    for (int d = 0; d < a->n_dev; ++d)
      if (!a->xin[d]) return fail(bt::ERR_INPUT, "null inbox of device %d", d);
    if (!bt::mlp_xdev_supported(*a))
      return fail(bt::ERR_INPUT, "multi-device step: E_total in {4,8,16} over 2/4/8 devices in equal blocks, "
                                 "micro-batch 4, one Sequential/Tree(2) variant");
    if (!a->replicas || !a->est_fanin || !a->rng || !a->stat_mean || !a->stat_count || !a->losses || !a->flags)
      return fail(bt::ERR_INPUT, "null device pointer in bt_mlp_args");
    return 0;
  }
  if (a->fuse_reduce && a->E != a->E_total)
    return fail(bt::ERR_INPUT, "fused allreduce needs every EST local (E == E_total)");
  if (a->fuse_reduce && !bt::mlp_fused_fits(*a))
    return fail(bt::ERR_INPUT, "%d ESTs do not fit the fused step's shared memory; use grads-only + bt_reduce_update",
                a->E_total);
  if (!a->fuse_reduce && a->K != 1) return fail(bt::ERR_INPUT, "grads-only mode runs one mini-batch");
  if (a->comm_fanin < 0 || a->comm_fanin == 1) return fail(bt::ERR_CONFIG, "bad allreduce fanin %d", a->comm_fanin);
  if (a->est_fanin_uniform < 0 || a->est_fanin_uniform == 2)
    return fail(bt::ERR_CONFIG, "bad est_fanin_uniform %d", a->est_fanin_uniform);
  if (!a->rows && (!a->dataset || !a->lists || a->spe < 1))
    return fail(bt::ERR_INPUT, "need either explicit rows or dataset+lists+spe");
  if (!a->replicas || !a->est_fanin || !a->rng || !a->stat_mean || !a->stat_count || !a->grads || !a->losses ||
      !a->flags)
    return fail(bt::ERR_INPUT, "null device pointer in bt_mlp_args");
  if (a->fuse_reduce && (a->E + a->est_per_cta - 1) / a->est_per_cta > 1 && !a->bar)
    return fail(bt::ERR_INPUT, "multi-CTA fused step needs a barrier word");
  return 0;
}

int bt_mlp_fused_fits(const bt_mlp_args* args) { return args && bt::mlp_fused_fits(*args) ? 1 : 0; }

int bt_mlp_step(const bt_mlp_args* args, void* stream) {
  int st = validate_mlp(args);
  if (st) return st;
  return done(bt::mlp_launch(*args, STREAM(stream)), "bt_mlp_step");
}

// Wait for the stream's work by polling an event (a spin, not a blocking wait): a blocking
// synchronisation costs tens of microseconds of wake-up latency, which is most of a short call.
static cudaError_t host_wait(cudaStream_t s) {
  static thread_local cudaEvent_t ev = nullptr;
  static thread_local int ev_dev = -1;
  int dev = 0;
  cudaGetDevice(&dev);
  if (!ev || ev_dev != dev) {
    if (cudaEventCreateWithFlags(&ev, cudaEventDisableTiming) != cudaSuccess) return cudaGetLastError();
    ev_dev = dev;
  }
  cudaError_t e = cudaEventRecord(ev, s);
  if (e != cudaSuccess) return e;
  while ((e = cudaEventQuery(ev)) == cudaErrorNotReady) {
  }
  return e;
}

// BT_HOST_SIGNAL=0: always copy the results back and synchronise the stream (measurements, tests).
static bool host_signal_enabled() {
  static const int on = [] {
    const char* e = getenv("BT_HOST_SIGNAL");
    return (e && strcmp(e, "0") == 0) ? 0 : 1;
  }();
  return on != 0;
}
// The host signal of bt_mlp_run: a mapped pinned done word per host thread, bumped per call.
static uint32_t* host_done_word(uint32_t** dev) {
  static thread_local uint32_t* w = nullptr;
  static thread_local uint32_t* wd = nullptr;
  if (!w) {
    void* p = nullptr;
    void* d = nullptr;
    if (cudaHostAlloc(&p, 64, cudaHostAllocPortable | cudaHostAllocMapped) != cudaSuccess ||
        cudaHostGetDevicePointer(&d, p, 0) != cudaSuccess) {
      if (p) cudaFreeHost(p);
      cudaGetLastError();
      return nullptr;
    }
    w = (uint32_t*)p;
    wd = (uint32_t*)d;
    *(volatile uint32_t*)w = 0;
  }
  *dev = wd;
  return w;
}
// device-accessible address of pinned host memory (null when p is not pinned); the last answer is cached
static void* mapped_ptr(void* p) {
  // a few recent (host, device) pairs: the result block and the sampler's staging buffers alternate
  static thread_local void* host[4] = {nullptr, nullptr, nullptr, nullptr};
  static thread_local void* devp[4] = {nullptr, nullptr, nullptr, nullptr};
  static thread_local unsigned next = 0;
  for (int i = 0; i < 4; ++i)
    if (host[i] == p && p) return devp[i];
  cudaPointerAttributes at;
  if (cudaPointerGetAttributes(&at, p) != cudaSuccess) {
    cudaGetLastError();
    return nullptr;
  }
  if (at.type != cudaMemoryTypeHost || !at.devicePointer) return nullptr;
  const unsigned i = next++ & 3;
  host[i] = p;
  devp[i] = at.devicePointer;
  return devp[i];
}

struct RunWait {  // how bt_mlp_run's results arrive: a host signal (seq on *done) or the stream
  volatile uint32_t* done = nullptr;
  uint32_t seq = 0;
};

// Everything of bt_mlp_run but the host wait: the launch and the results' way back, queued on s.  In the
// one-copy layout with pinned host buffers the compact build's epilogue writes the losses and status words
// into host memory itself and signals a done word (no copy, no stream synchronisation); otherwise one or
// two device-to-host copies follow the launch.
static int mlp_run_enqueue(const bt_mlp_args* args, double* losses_host, int32_t* status_host, cudaStream_t s,
                           RunWait* w) {
  const size_t lbytes = sizeof(double) * (size_t)args->K * args->E_total;
  // status_host == NULL: the status block directly follows the losses in device memory, and ONE copy
  // brings both (status words at the tail of losses_host)
  const bool one_copy = !status_host && losses_host && (const char*)args->flags == (const char*)args->losses + lbytes;
  if (!status_host && !one_copy)
    return fail(bt::ERR_INPUT, "bt_mlp_run needs a status buffer (or the status block right after the losses)");
  w->done = nullptr;
  if (one_copy && args->n_dev <= 1 && host_signal_enabled()) {
    void* dev_out = mapped_ptr(losses_host);
    uint32_t* dw_dev = nullptr;
    uint32_t* dw = dev_out ? host_done_word(&dw_dev) : nullptr;
    if (dw) {
      static thread_local uint32_t seq = 0;
      const bt::MlpHostSignal hs{(double*)dev_out, dw_dev, ++seq};
      bool signaled = false;
      const int st = bt::mlp_launch(*args, s, nullptr, &hs, &signaled);
      if (st) return done(st, "bt_mlp_run");
      if (signaled) {
        w->done = dw;
        w->seq = hs.seq;
        return 0;
      }
      // (the generic build ran: copy back below)
      if (cudaMemcpyAsync(losses_host, args->losses, lbytes + 4 * sizeof(int32_t), cudaMemcpyDeviceToHost, s) !=
          cudaSuccess)
        return cuda_fail("bt_mlp_run losses + status");
      return 0;
    }
  }
  const int st = bt::mlp_launch(*args, s);
  if (st) return done(st, "bt_mlp_run");
  if (one_copy) {
    if (cudaMemcpyAsync(losses_host, args->losses, lbytes + 4 * sizeof(int32_t), cudaMemcpyDeviceToHost, s) !=
        cudaSuccess)
      return cuda_fail("bt_mlp_run losses + status");
  } else {
    if (losses_host && cudaMemcpyAsync(losses_host, args->losses, lbytes, cudaMemcpyDeviceToHost, s) != cudaSuccess)
      return cuda_fail("bt_mlp_run losses");
    if (cudaMemcpyAsync(status_host, args->flags, 4 * sizeof(int32_t), cudaMemcpyDeviceToHost, s) != cudaSuccess)
      return cuda_fail("bt_mlp_run status");
  }
  return 0;
}

// Wait for the results: spin on the done word (checking the stream now and then, so a failed or
// non-signalling launch is reported instead of waited on forever), or poll the stream's event.
static int mlp_run_wait(cudaStream_t s, const RunWait& w, const char* what) {
  if (!w.done) return host_wait(s) == cudaSuccess ? 0 : cuda_fail(what);
  for (uint32_t it = 1;; ++it) {
    if (*w.done == w.seq) break;
    if ((it & 255) == 0) {
      const cudaError_t q = cudaStreamQuery(s);
      if (q == cudaSuccess) {
        if (*w.done == w.seq) break;
        return fail(bt::ERR_CUDA, "%s: the launch completed without signalling its results", what);
      }
      if (q != cudaErrorNotReady) return cuda_fail(what);
    }
  }
  __atomic_thread_fence(__ATOMIC_ACQUIRE);  // the results the done word published
  return 0;
}

int bt_mlp_run(const bt_mlp_args* args, double* losses_host, int32_t* status_host, void* stream) {
  int st = validate_mlp(args);
  if (st) return st;
  cudaStream_t s = STREAM(stream);
  RunWait w;
  st = mlp_run_enqueue(args, losses_host, status_host, s, &w);
  if (st) return st;
  st = mlp_run_wait(s, w, "bt_mlp_run sync");
  if (st) return st;
  g_err[0] = 0;
  return 0;
}

static bool lists_zero_copy() {  // BT_LISTS_ZC=0: copy the lists to the device before the launch (A/B)
  static const int on = [] {
    const char* e = getenv("BT_LISTS_ZC");
    return (e && strcmp(e, "0") == 0) ? 0 : 1;
  }();
  return on != 0;
}
// Staging buffers whose device copy may still be queued: (buffer, device, event after the copy).
struct StageCopy {
  const void* host;
  int dev;
  cudaEvent_t ev;
  bool pending;
};
static StageCopy g_stage[8];
static int stage_copy_wait(const void* host) {
  for (auto& c : g_stage)
    if (c.host == host && c.pending) {
      c.pending = false;
      if (cudaEventSynchronize(c.ev) != cudaSuccess) return cuda_fail("bt_mlp_run_sampled staging reuse");
    }
  return 0;
}
static void stage_copy_record(const void* host, cudaStream_t s) {
  int dev = 0;
  cudaGetDevice(&dev);
  StageCopy* slot = nullptr;
  for (auto& c : g_stage)
    if (c.host == host && c.dev == dev) slot = &c;
  if (!slot)
    for (auto& c : g_stage)
      if (!c.host || !c.pending) {
        if (c.host && c.ev) cudaEventDestroy(c.ev);
        c = StageCopy{host, dev, nullptr, false};
        slot = &c;
        break;
      }
  if (!slot) {  // every slot busy: wait for the stream instead (never observed: two buffers per pipeline)
    cudaStreamSynchronize(s);
    return;
  }
  if (!slot->ev && cudaEventCreateWithFlags(&slot->ev, cudaEventDisableTiming) != cudaSuccess) {
    cudaGetLastError();
    slot->ev = nullptr;
    cudaStreamSynchronize(s);
    return;
  }
  if (cudaEventRecord(slot->ev, s) != cudaSuccess) {
    cudaGetLastError();
    cudaStreamSynchronize(s);
    return;
  }
  slot->pending = true;
}

int bt_stage_wait(const void* stage_host) { return stage_copy_wait(stage_host); }

int bt_mlp_run_sampled(const bt_mlp_args* args, uint64_t seed, int64_t dataset_n, int32_t shuffle,
                       int64_t first_epoch, int32_t n_epochs, int32_t* stage_host, int32_t* lists_dev,
                       double* losses_host, int32_t* status_host, void* stream) {
  if (!args || !stage_host || !lists_dev) return fail(bt::ERR_INPUT, "bt_mlp_run_sampled: null pointer");
  if (n_epochs < 1 || first_epoch < 0) return fail(bt::ERR_INPUT, "bt_mlp_run_sampled: %d epochs", n_epochs);
  const int32_t workers = args->E_total, micro = args->B;
  if (workers < 1 || micro < 1 || args->spe < 1 || dataset_n / ((int64_t)workers * micro) != args->spe)
    return fail(bt::ERR_CONFIG, "bt_mlp_run_sampled: steps per epoch %lld do not match the dataset", (long long)args->spe);
  // the launch's epochs must be the ones staged
  if (args->step0 / args->spe < first_epoch ||
      (args->step0 + args->K - 1) / args->spe >= first_epoch + n_epochs)
    return fail(bt::ERR_INPUT, "bt_mlp_run_sampled: epochs [%lld, +%d) do not cover the launch",
                (long long)first_epoch, n_epochs);
  bt_mlp_args a = *args;
  a.lists = lists_dev;
  a.epoch_base = first_epoch;
  int st = validate_mlp(&a);
  if (st) return st;
  const size_t per = (size_t)workers * (size_t)(args->spe * micro);
  st = stage_copy_wait(stage_host);  // a previous call's copy out of this staging buffer has finished
  if (st) return st;
  for (int32_t k = 0; k < n_epochs; ++k) {  // the sampler's host work (sampling.py:63-82), then one H2D copy
    st = bt_host_epoch_indices(seed, (uint64_t)(first_epoch + k), dataset_n, workers, micro, shuffle,
                               stage_host + (size_t)k * per);
    if (st) return st;
  }
  // (Overlapping this host work with the launch latency -- the stream held on a pinned gate word while
  // the copy and launch are queued, then opened -- was measured slower: +15 us per call, the device's
  // poll of host memory costing more than the ~8 us of Fisher-Yates it hides.)
  cudaStream_t s = STREAM(stream);
  const size_t lbytes = sizeof(int32_t) * per * n_epochs;
  // Zero-copy: the launch reads this call's index lists straight from the pinned staging buffer (the
  // compact build loads them once, in its prologue, beside its other global loads: one PCIe round trip
  // instead of a DMA copy the launch has to wait for); the device copy that later calls of the same
  // epochs use is queued AFTER the launch, off the path to the results (the caller re-fills this staging
  // buffer only after that copy: bt_stage_reuse_wait).
  int32_t* zc = lists_zero_copy() ? (int32_t*)mapped_ptr(stage_host) : nullptr;
  RunWait w;
  if (zc) {
    a.lists = zc;
    st = mlp_run_enqueue(&a, losses_host, status_host, s, &w);
    if (st) return st;
    if (cudaMemcpyAsync(lists_dev, stage_host, lbytes, cudaMemcpyHostToDevice, s) != cudaSuccess)
      return cuda_fail("bt_mlp_run_sampled lists");
    stage_copy_record(stage_host, s);
  } else {
    if (cudaMemcpyAsync(lists_dev, stage_host, lbytes, cudaMemcpyHostToDevice, s) != cudaSuccess)
      return cuda_fail("bt_mlp_run_sampled lists");
    st = mlp_run_enqueue(&a, losses_host, status_host, s, &w);
    if (st) return st;
  }
  st = mlp_run_wait(s, w, "bt_mlp_run_sampled sync");
  if (st) return st;
  g_err[0] = 0;
  return 0;
}

int bt_mlp_run_group(const bt_mlp_args* const* args, const int32_t* devices, void* const* streams, int32_t n,
                     double* const* losses_host, int32_t* const* status_host) {
  if (n < 1 || n > BT_MAX_XDEV) return fail(bt::ERR_INPUT, "group of %d launches", n);
  int cur = 0;
  cudaGetDevice(&cur);
  for (int i = 0; i < n; ++i) {  // validate everything before anything runs: the launches wait on each other
    const int st = validate_mlp(args[i]);
    if (st) return st;
    if (!status_host[i]) return fail(bt::ERR_INPUT, "bt_mlp_run_group needs status buffers");
  }
  int rc = 0;
  for (int i = 0; i < n && !rc; ++i) {  // every device's launch is queued before any host wait
    if (cudaSetDevice(devices[i]) != cudaSuccess) rc = cuda_fail("bt_mlp_run_group set device");
    else rc = done(bt::mlp_launch(*args[i], STREAM(streams[i])), "bt_mlp_run_group");
  }
  for (int i = 0; i < n && !rc; ++i) {
    cudaStream_t s = STREAM(streams[i]);
    cudaSetDevice(devices[i]);
    if (losses_host[i] && cudaMemcpyAsync(losses_host[i], args[i]->losses,
                                          sizeof(double) * (size_t)args[i]->K * args[i]->E_total,
                                          cudaMemcpyDeviceToHost, s) != cudaSuccess)
      rc = cuda_fail("bt_mlp_run_group losses");
    else if (cudaMemcpyAsync(status_host[i], args[i]->flags, 4 * sizeof(int32_t), cudaMemcpyDeviceToHost, s) !=
             cudaSuccess)
      rc = cuda_fail("bt_mlp_run_group status");
  }
  for (int i = 0; i < n; ++i) {  // (also after a failed launch: no queued work outlives the call)
    cudaSetDevice(devices[i]);
    if (cudaStreamSynchronize(STREAM(streams[i])) != cudaSuccess && !rc) rc = cuda_fail("bt_mlp_run_group sync");
  }
  cudaSetDevice(cur);
  if (!rc) g_err[0] = 0;
  return rc;
}

int bt_mlp_step_profiled(const bt_mlp_args* args, uint64_t* timing_dev, void* stream) {
  int st = validate_mlp(args);
  if (st) return st;
  return done(bt::mlp_launch(*args, STREAM(stream), (unsigned long long*)timing_dev), "bt_mlp_step_profiled");
}

int bt_fwd_bwd_mlp_f64(const double* params_dev, const double* rows_dev, int32_t E, int32_t est_base,
                       int32_t E_total, int32_t B, const int32_t* est_fanin_dev, double rate, int64_t rank_override,
                       uint64_t* rng_io_dev, double* stat_mean_io_dev, uint64_t* stat_count_io_dev,
                       double* losses_out_dev, double* grads_out_dev, int32_t* flags_dev, void* stream) {
  bt_mlp_args a;
  memset(&a, 0, sizeof a);
  a.E = E;
  a.est_base = est_base;
  a.E_total = E_total;
  a.B = B;
  a.X = 1;
  a.K = 1;
  a.fuse_reduce = 0;
  a.est_per_cta = bt_mlp_pick_est_per_cta(E, B);
  if ((int64_t)a.est_per_cta * B > 256) a.est_per_cta = 256 / (B > 0 ? B : 1);
  a.rank_override = rank_override;
  a.rate = rate;
  a.replicas = (double*)params_dev;
  a.est_fanin = est_fanin_dev;
  a.rng = rng_io_dev;
  a.stat_mean = stat_mean_io_dev;
  a.stat_count = stat_count_io_dev;
  a.grads = grads_out_dev;
  a.losses = losses_out_dev;
  a.rows = rows_dev;
  a.flags = flags_dev;
  return bt_mlp_step(&a, stream);
}

// ------------------------------------------------------ tensor-core GEMM
int bt_gemm_bf16_ex(const void* a_dev, const void* b_dev, void* c_dev, int32_t batch, int32_t M, int32_t N, int32_t K,
                    int64_t stride_a, int64_t stride_b, int64_t stride_c, int32_t out_dtype, const float* bias_dev,
                    int32_t mn_major, int32_t grid, void* stream) {
  if (!a_dev || !b_dev || !c_dev) return fail(bt::ERR_INPUT, "null pointer");
  if (mn_major < 0 || mn_major > 2) return fail(bt::ERR_INPUT, "mn_major %d: 0, 1 or 2", mn_major);
  if (batch < 1 || M <= 0 || N <= 0 || K <= 0 || N % 8 || (mn_major == 1 ? M % 8 : K % 8))
    return fail(bt::ERR_INPUT, "gemm shape %dx%dx%d x%d: need N %% 8 == 0 and %s %% 8 == 0 (16-byte TMA strides)", M,
                N, K, batch, mn_major == 1 ? "M" : "K");
  if (((uintptr_t)a_dev | (uintptr_t)b_dev | (uintptr_t)c_dev | (uintptr_t)bias_dev) & 15)
    return fail(bt::ERR_INPUT, "gemm operands must be 16-byte aligned");
  if (batch == 1) {
    stride_a = (int64_t)M * K;
    stride_b = (int64_t)N * K;
    stride_c = (int64_t)M * N;
  }
  if (stride_c == 0) stride_c = (int64_t)M * N;
  if (stride_a < (int64_t)M * K || stride_b < (int64_t)N * K || stride_c < (int64_t)M * N ||
      (stride_a | stride_b | stride_c) % 8)
    return fail(bt::ERR_INPUT, "gemm batch strides must cover a matrix and be multiples of 8 elements");
  if (out_dtype != 0 && out_dtype != 1) return fail(bt::ERR_INPUT, "gemm out_dtype must be 0 (f32) or 1 (bf16)");
  bt::GemmEpi epi{};
  epi.kind = bias_dev ? bt::EPI_BIAS : bt::EPI_STORE;
  epi.bias = bias_dev;
  return done(bt::gemm_bf16_launch_any(a_dev, b_dev, c_dev, batch, M, N, K, stride_a, stride_b, stride_c, out_dtype,
                                       grid, epi, mn_major, STREAM(stream)),
              "bt_gemm_bf16");
}
int bt_gemm_conv(int32_t wgrad, const void* x_dev, int32_t xN, int32_t xH, int32_t xW, int32_t Ci, int32_t Ho,
                 int32_t Wo, int32_t KH, int32_t KW, int32_t stride, int32_t pad, const void* other_dev, void* c_dev,
                 int32_t Co, int32_t batch, int32_t rows_per_batch, int64_t stride_c, int32_t out_dtype, void* stream) {
  if (!x_dev || !other_dev || !c_dev) return fail(bt::ERR_INPUT, "null pointer");
  if (Ci % 64 || Ci > 4096 || Co % 8 || Co < 8 || xN < 1 || xH < 1 || xW < 1 || Ho < 1 || Wo < 1 || KH < 1 || KW < 1 ||
      stride < 1 || stride > 8 || pad < 0 || pad > 16 || (out_dtype != 0 && out_dtype != 1))
    return fail(bt::ERR_INPUT, "bt_gemm_conv geometry (Ci %% 64 == 0, Co %% 8 == 0)");
  if (wgrad && (batch < 1 || rows_per_batch < 64 || rows_per_batch % 64 || (int64_t)batch * rows_per_batch !=
                (int64_t)xN * Ho * Wo || stride_c < (int64_t)Co * KH * KW * Ci || stride_c % 8))
    return fail(bt::ERR_INPUT, "bt_gemm_conv wgrad: rows_per_batch %% 64 == 0, batches covering the output");
  if (((uintptr_t)x_dev | (uintptr_t)other_dev | (uintptr_t)c_dev) & 15)
    return fail(bt::ERR_INPUT, "operands must be 16-byte aligned");
  return done(bt::gemm_conv_launch(wgrad, x_dev, xN, xH, xW, Ci, Ho, Wo, KH, KW, stride, pad, other_dev, c_dev, Co,
                                   batch, rows_per_batch, stride_c, out_dtype, STREAM(stream)),
              "bt_gemm_conv");
}

int bt_gemm_bf16_tn_ex(const void* a_dev, const void* b_dev, void* c_dev, int32_t batch, int32_t M, int32_t N,
                       int32_t K, int64_t stride_a, int64_t stride_b, int64_t stride_c, int32_t out_dtype,
                       const float* bias_dev, int32_t grid, void* stream) {
  return bt_gemm_bf16_ex(a_dev, b_dev, c_dev, batch, M, N, K, stride_a, stride_b, stride_c, out_dtype, bias_dev, 0,
                         grid, stream);
}

int bt_gemm_bf16_tn_batched(const void* a_dev, const void* b_dev, void* c_dev, int32_t batch, int32_t M, int32_t N,
                            int32_t K, int64_t stride_a, int64_t stride_b, int32_t out_dtype, int32_t grid,
                            void* stream) {
  return bt_gemm_bf16_tn_ex(a_dev, b_dev, c_dev, batch, M, N, K, stride_a, stride_b, (int64_t)M * N, out_dtype,
                            nullptr, grid, stream);
}

int bt_gemm_bf16_tn(const void* a_dev, const void* b_dev, void* c_dev, int32_t M, int32_t N, int32_t K,
                    int32_t out_dtype, int32_t grid, void* stream) {
  return bt_gemm_bf16_tn_batched(a_dev, b_dev, c_dev, 1, M, N, K, 0, 0, out_dtype, grid, stream);
}

int bt_gemm_bf16_ffn(const void* a_dev, const void* b_dev, void* c_dev, int32_t M, int32_t N, int32_t K, int32_t kind,
                     const float* bias_dev, const void* aux_dev, void* out2_dev, uint64_t seed, int64_t step,
                     int32_t est_base, int32_t Te, float p, int32_t grid, void* stream) {
  return bt_gemm_bf16_ffn_cs(a_dev, b_dev, c_dev, M, N, K, kind, bias_dev, aux_dev, out2_dev, nullptr, seed, step,
                             est_base, Te, p, grid, stream);
}
int bt_gemm_bf16_ffn_cs(const void* a_dev, const void* b_dev, void* c_dev, int32_t M, int32_t N, int32_t K,
                        int32_t kind, const float* bias_dev, const void* aux_dev, void* out2_dev, float* colpart_dev,
                        uint64_t seed, int64_t step, int32_t est_base, int32_t Te, float p, int32_t grid,
                        void* stream) {
  if (!a_dev || !b_dev || !c_dev) return fail(bt::ERR_INPUT, "null pointer");
  if (M <= 0 || N <= 0 || K <= 0 || M % 128 || N % 128 || K % 64)
    return fail(bt::ERR_INPUT, "gemm shape %dx%dx%d: need M %% 128 == 0, N %% 128 == 0, K %% 64 == 0", M, N, K);
  const bool b_mn = (kind & BT_GEMM_B_MN) != 0;  // B stored [K][N] (the weights as stored: no transposed copy)
  kind &= ~BT_GEMM_B_MN;
  if (kind != bt::EPI_FFN_FWD && kind != bt::EPI_FFN_BWD) return fail(bt::ERR_INPUT, "bad epilogue kind %d", kind);
  if (kind == bt::EPI_FFN_FWD && (!bias_dev || !out2_dev)) return fail(bt::ERR_INPUT, "FFN_FWD needs bias and out2");
  if (kind == bt::EPI_FFN_BWD && !aux_dev) return fail(bt::ERR_INPUT, "FFN_BWD needs the pre-activations");
  if (Te < 1 || M % Te || !(p >= 0.f && p < 1.f)) return fail(bt::ERR_CONFIG, "bad Te %d / dropout %g", Te, (double)p);
  if (((uintptr_t)a_dev | (uintptr_t)b_dev | (uintptr_t)c_dev | (uintptr_t)aux_dev | (uintptr_t)out2_dev) & 15)
    return fail(bt::ERR_INPUT, "gemm operands must be 16-byte aligned");
  bt::GemmEpi epi{};
  epi.kind = kind;
  epi.bias = bias_dev;
  epi.aux = (const __nv_bfloat16*)aux_dev;
  epi.out2 = (__nv_bfloat16*)out2_dev;
  epi.seed = seed;
  epi.step = step;
  epi.est_base = est_base;
  epi.Te = Te;
  epi.p = p;
  if (colpart_dev && kind != bt::EPI_FFN_BWD) return fail(bt::ERR_INPUT, "column partials are an FFN_BWD output");
  if ((uintptr_t)colpart_dev & 7) return fail(bt::ERR_INPUT, "column partials must be 8-byte aligned");
  epi.colpart = colpart_dev;
  return done(bt::gemm_bf16_launch_any(a_dev, b_dev, c_dev, 1, M, N, K, (int64_t)M * K, (int64_t)N * K,
                                       (int64_t)M * N, 1, grid, epi, b_mn ? 2 : 0, STREAM(stream)),
              "bt_gemm_bf16_ffn");
}

// ------------------------------------------ per-EST FFN step (C4 slice)
static int ffn_check(int E, int Te, int D) {
  if (E < 1 || Te < 1 || D < 1) return fail(bt::ERR_INPUT, "ffn shape E=%d Te=%d D=%d", E, Te, D);
  return 0;
}
int bt_ffn_data(uint64_t seed, int64_t step, int32_t est_base, int32_t E, int32_t Te, int32_t D, void* x_dev,
                float* target_dev, void* stream) {
  if (int st = ffn_check(E, Te, D)) return st;
  return done(bt::ffn_data_launch(seed, step, est_base, E, Te, D, x_dev, target_dev, STREAM(stream)), "bt_ffn_data");
}
int bt_ffn_fwd_act(const float* h_dev, const float* b1_dev, uint64_t seed, int64_t step, int32_t est_base, int32_t E,
                   int32_t Te, int32_t F, float p, void* hpre_dev, void* d_dev, void* stream) {
  if (int st = ffn_check(E, Te, F)) return st;
  if (!(p >= 0.f && p < 1.f)) return fail(bt::ERR_CONFIG, "dropout rate %g not in [0, 1)", (double)p);
  return done(bt::ffn_fwd_act_launch(h_dev, b1_dev, seed, step, est_base, E, Te, F, p, hpre_dev, d_dev,
                                     STREAM(stream)),
              "bt_ffn_fwd_act");
}
int bt_ffn_out(const float* y_dev, const float* b2_dev, const float* target_dev, int32_t E, int32_t Te, int32_t D,
               void* dy_dev, float* partials_dev, float* loss_dev, void* stream) {
  if (int st = ffn_check(E, Te, D)) return st;
  return done(bt::ffn_out_launch(y_dev, b2_dev, target_dev, E, Te, D, dy_dev, partials_dev, loss_dev, STREAM(stream)),
              "bt_ffn_out");
}
int bt_ffn_bwd_act(const float* dd_dev, const void* hpre_dev, uint64_t seed, int64_t step, int32_t est_base, int32_t E,
                   int32_t Te, int32_t F, float p, void* dh_dev, void* stream) {
  if (int st = ffn_check(E, Te, F)) return st;
  if (!(p >= 0.f && p < 1.f)) return fail(bt::ERR_CONFIG, "dropout rate %g not in [0, 1)", (double)p);
  return done(bt::ffn_bwd_act_launch(dd_dev, hpre_dev, seed, step, est_base, E, Te, F, p, dh_dev, STREAM(stream)),
              "bt_ffn_bwd_act");
}
int bt_colsum_bf16(const void* in_dev, int32_t E, int32_t R, int32_t C, float* out_dev, float* scratch_dev,
                   void* stream) {
  if (int st = ffn_check(E, R, C)) return st;
  return done(bt::colsum_bf16_launch(in_dev, E, R, C, out_dev, scratch_dev, STREAM(stream)), "bt_colsum_bf16");
}
int bt_transpose_to_bf16(const void* in_dev, int32_t in_f32, int32_t E, int32_t R, int32_t C, void* out_dev,
                         void* stream) {
  if (int st = ffn_check(E, R, C)) return st;
  return done(bt::transpose_launch(in_dev, in_f32, E, R, C, out_dev, STREAM(stream)), "bt_transpose_to_bf16");
}
int bt_cast_f32_bf16(const float* in_dev, int64_t n, void* out_dev, void* stream) {
  if (n < 0) return fail(bt::ERR_INPUT, "negative length");
  return done(bt::cast_f32_bf16_launch(in_dev, n, out_dev, STREAM(stream)), "bt_cast_f32_bf16");
}

// ------------------------------------------------------------- device: L2
int bt_reduce_update(const bt_reduce_args* a, void* stream) {
  if (!a) return fail(bt::ERR_INPUT, "null args");
  if (a->dtype != BT_DTYPE_F64 && a->dtype != BT_DTYPE_F32) return fail(bt::ERR_INPUT, "bad dtype %d", a->dtype);
  if (a->E < 1) return fail(bt::ERR_INPUT, "need at least one gradient replica");
  if (a->grads_ld == 0 && a->E > BT_MAX_TABLE)
    return fail(bt::ERR_INPUT, "pointer-table mode holds at most %d contributions", BT_MAX_TABLE);
  if (a->fanin < 0 || a->fanin == 1) return fail(bt::ERR_CONFIG, "bad fanin %d", a->fanin);
  if (a->n < 0) return fail(bt::ERR_INPUT, "negative length");
  if (a->nout < 0 || a->nout > BT_MAX_REPLICA_OUT) return fail(bt::ERR_INPUT, "nout outside [0, 8]");
  if (a->mode < BT_REDUCE_UPDATE || a->mode > BT_REDUCE_APPLY_ADAM) return fail(bt::ERR_INPUT, "bad mode %d", a->mode);
  if (a->mode == BT_REDUCE_MEAN_CHECK && !a->flags) return fail(bt::ERR_INPUT, "MEAN_CHECK needs the flags");
  if ((a->mode == BT_REDUCE_APPLY_SGD || a->mode == BT_REDUCE_APPLY_ADAM) &&
      (!a->stage || !a->param || !a->vel || !a->vel_out || !a->flags))
    return fail(bt::ERR_INPUT, "APPLY needs stage, param, vel and flags");
  if (a->mode == BT_REDUCE_APPLY_ADAM && (!a->vel2 || !a->vel2_out))
    return fail(bt::ERR_INPUT, "Adam needs the second-moment buffers");
  if (a->ngate < 0 || (a->ngate > 0 && !a->gate)) return fail(bt::ERR_INPUT, "bad gate table");
  if (a->divisor < 0) return fail(bt::ERR_INPUT, "negative divisor");
  const bool upd = a->mode == BT_REDUCE_UPDATE || a->mode == BT_REDUCE_ADAM;
  if (!a->param_out || (upd && (!a->param || !a->vel || !a->vel_out || !a->flags)))
    return fail(bt::ERR_INPUT, "null buffer");
  if (a->mode == BT_REDUCE_ADAM) {
    if (!a->vel2 || !a->vel2_out) return fail(bt::ERR_INPUT, "Adam needs the second-moment buffers");
    for (int r = 0; r < a->nout; ++r)
      if (!a->extra_vel2_out[r]) return fail(bt::ERR_INPUT, "Adam replica outputs need extra_vel2_out");
    if (!(a->eps > 0) || !(a->beta2 >= 0 && a->beta2 < 1) || !(a->mu >= 0 && a->mu < 1) || !(a->bc1 > 0) ||
        !(a->bc2 > 0))
      return fail(bt::ERR_CONFIG, "Adam hyper-parameters: 0 <= beta1, beta2 < 1, eps > 0, bias corrections > 0");
  }
  return done(bt::reduce_launch(*a, STREAM(stream)), "bt_reduce_update");
}

int bt_sgd_step_f64(const double* params_dev, const double* vel_dev, const double* grads_dev, int64_t n, double lr,
                    double mu, double* params_out_dev, double* vel_out_dev, int32_t* flags_dev, void* stream) {
  if (n < 0) return fail(bt::ERR_INPUT, "negative length");
  if (n == 0) return 0;
  return done(bt::sgd_launch(params_dev, vel_dev, grads_dev, n, lr, mu, params_out_dev, vel_out_dev, flags_dev,
                             STREAM(stream)),
              "bt_sgd_step_f64");
}

// ------------------------------------------------------------- device: L3
int bt_make_dataset(uint64_t seed, int64_t n, int32_t dim, double* out_dev, void* stream) {
  if (n < 0 || dim < 0) return fail(bt::ERR_INPUT, "bad dataset shape");
  if (n == 0) return 0;
  return done(bt::make_dataset_launch(seed, n, dim, out_dev, STREAM(stream)), "bt_make_dataset");
}

int bt_jitter_gather(const double* dataset_dev, const int32_t* lists_dev, int32_t E, int32_t est_base,
                     int32_t E_total, int32_t B, int64_t spe, uint64_t seed, int64_t epoch, int64_t local,
                     double jitter, double* rows_out_dev, void* stream) {
  if (E < 1 || B < 1 || est_base < 0 || est_base + E > E_total || local < 0 || local >= spe)
    return fail(bt::ERR_INPUT, "bad jitter_gather shape");
  return done(bt::jitter_gather_launch(dataset_dev, lists_dev, E, est_base, E_total, B, spe, seed, epoch, local,
                                       jitter, rows_out_dev, STREAM(stream)),
              "bt_jitter_gather");
}

int bt_dropout_mask(uint64_t state, int64_t rows, int32_t units, double rate, double* out_dev, void* stream) {
  if (rows < 0 || units < 0) return fail(bt::ERR_INPUT, "bad mask shape");
  if (rows * units == 0) return 0;
  return done(bt::dropout_mask_launch(state, rows, units, rate, out_dev, STREAM(stream)), "bt_dropout_mask");
}

// ------------------------------------------------------------- device: L4
int bt_replica_check(const void* const* ptrs, int32_t R, int64_t nbytes, int32_t* flags_dev, void* stream) {
  if (R < 1 || R > 64) return fail(bt::ERR_INPUT, "replica count %d outside [1, 64]", R);
  if (nbytes % 8) return fail(bt::ERR_INPUT, "replica size must be a multiple of 8 bytes");
  if (R == 1 || nbytes == 0) return 0;
  return done(bt::replica_check_launch(ptrs, R, nbytes, flags_dev, STREAM(stream)), "bt_replica_check");
}

int bt_est_slot_copy(void* const* dst, const void* const* src, const int64_t* bytes, int32_t count, void* stream) {
  if (count < 0 || count > 64) return fail(bt::ERR_INPUT, "slot copy count %d outside [0, 64]", count);
  if (count == 0) return 0;
  return done(bt::slot_copy_launch(dst, src, bytes, count, STREAM(stream)), "bt_est_slot_copy");
}

int bt_allgather_params(int32_t dtype, const void* src_dev, void* const* dst_dev, int32_t ndst, int64_t n,
                        void* stream) {
  if (ndst < 0 || ndst > 64) return fail(bt::ERR_INPUT, "ndst outside [0, 64]");
  const int64_t es = dtype == BT_DTYPE_F64 ? 8 : 4;
  const void* srcs[64];
  int64_t bytes[64];
  for (int i = 0; i < ndst; ++i) {
    srcs[i] = src_dev;
    bytes[i] = n * es;
  }
  return bt_est_slot_copy(dst_dev, srcs, bytes, ndst, stream);
}

int bt_memcpy_async(void* dst, const void* src, int64_t nbytes, void* stream) {
  if (nbytes < 0) return fail(bt::ERR_INPUT, "negative byte count");
  if (nbytes == 0) return 0;
  if (cudaMemcpyAsync(dst, src, (size_t)nbytes, cudaMemcpyDefault, STREAM(stream)) != cudaSuccess)
    return cuda_fail("bt_memcpy_async");
  return 0;
}

int bt_fnv1a64_chunks(const void* data_dev, int64_t nbytes, int64_t chunk, uint64_t* out_dev, void* stream) {
  if (!data_dev || !out_dev || nbytes < 1 || chunk < 16 || chunk % 16) return fail(bt::ERR_INPUT, "fnv chunks");
  return done(bt::fnv_chunks_launch(data_dev, nbytes, chunk, out_dev, STREAM(stream)), "bt_fnv1a64_chunks");
}

int bt_l2_flush(void* buf_dev, int64_t bytes, uint32_t value, void* stream) {
  if (!buf_dev || bytes < 16 || ((uintptr_t)buf_dev & 15)) return fail(bt::ERR_INPUT, "l2 flush buffer");
  return done(bt::l2_flush_launch(buf_dev, bytes, value, STREAM(stream)), "bt_l2_flush");
}
int bt_flags_reset(int32_t* flags_dev, void* stream) {
  return done(bt::flags_reset_launch(flags_dev, STREAM(stream)), "bt_flags_reset");
}

int bt_step_status(const int32_t* flags_dev, int32_t* detail_out, int32_t* step_out, void* stream) {
  int32_t h[4];
  if (cudaMemcpyAsync(h, flags_dev, sizeof h, cudaMemcpyDeviceToHost, STREAM(stream)) != cudaSuccess)
    return cuda_fail("bt_step_status");
  if (cudaStreamSynchronize(STREAM(stream)) != cudaSuccess) return cuda_fail("bt_step_status sync");
  if (detail_out) *detail_out = h[bt::FLAG_DETAIL];
  if (step_out) *step_out = h[bt::FLAG_STEP];
  if (h[0] != 0) {
    snprintf(g_err, sizeof g_err, "device status %d (detail %d, step %d)", h[0], h[1], h[2]);
  }
  return h[0];
}

// ------------------------------------------------------------- multi-GPU
}  // extern "C"

// Driver entry points through the runtime (no link-time dependency on libcuda,
// so the library still loads on a GPU-less build host).
typedef int (*PFN_getAddressRange)(unsigned long long*, size_t*, unsigned long long);
typedef int (*PFN_streamWriteValue32)(void*, unsigned long long, unsigned int, unsigned int);
typedef int (*PFN_streamWaitValue32)(void*, unsigned long long, unsigned int, unsigned int);
template <typename F>
static F driver_fn(const char* name) {
  void* fn = nullptr;
  cudaDriverEntryPointQueryResult q;
  if (cudaGetDriverEntryPoint(name, &fn, cudaEnableDefault, &q) != cudaSuccess || q != cudaDriverEntryPointSuccess)
    return nullptr;
  return (F)fn;
}

extern "C" {

int bt_ipc_handle_size(void) { return (int)sizeof(cudaIpcMemHandle_t); }
int bt_ipc_get_handle(const void* dev_ptr, void* handle_out, int64_t* offset_out) {
  // An IPC handle names a whole cudaMalloc allocation; caching allocators hand
  // out sub-ranges, so return the handle of the base plus the byte offset.
  static PFN_getAddressRange range = driver_fn<PFN_getAddressRange>("cuMemGetAddressRange");
  unsigned long long base = (unsigned long long)dev_ptr;
  size_t size = 0;
  if (range && range(&base, &size, (unsigned long long)dev_ptr) != 0) return fail(bt::ERR_CUDA, "cuMemGetAddressRange");
  cudaIpcMemHandle_t h;
  if (cudaIpcGetMemHandle(&h, (void*)base) != cudaSuccess) return cuda_fail("cudaIpcGetMemHandle");
  memcpy(handle_out, &h, sizeof h);
  if (offset_out) *offset_out = (int64_t)((unsigned long long)dev_ptr - base);
  return 0;
}

// Stream-ordered cross-GPU signalling (no host barrier, no spinning kernel):
// write a 32-bit word (local or peer/IPC memory) when the stream reaches this
// point, and block a stream until a word is >= value.
int bt_stream_write_u32(void* dev_ptr, uint32_t value, void* stream) {
  static PFN_streamWriteValue32 fn = driver_fn<PFN_streamWriteValue32>("cuStreamWriteValue32");
  if (!fn) return fail(bt::ERR_CUDA, "cuStreamWriteValue32 unavailable");
  if (fn(stream, (unsigned long long)dev_ptr, value, 0 /*CU_STREAM_WRITE_VALUE_DEFAULT*/) != 0)
    return fail(bt::ERR_CUDA, "cuStreamWriteValue32 failed");
  return 0;
}
typedef int (*PFN_deviceGetAttribute)(int*, int, int);
int bt_stream_wait_u32_geq(void* dev_ptr, uint32_t value, void* stream) {
  static PFN_streamWaitValue32 fn = driver_fn<PFN_streamWaitValue32>("cuStreamWaitValue32");
  static PFN_deviceGetAttribute attr = driver_fn<PFN_deviceGetAttribute>("cuDeviceGetAttribute");
  if (!fn) return fail(bt::ERR_CUDA, "cuStreamWaitValue32 unavailable");
  // The wait is followed by reads of data other GPUs wrote to this one (peer stores, IPC): where
  // the device supports it, CU_STREAM_WAIT_VALUE_FLUSH makes those remote writes visible first.
  static int flush = -1;
  if (flush < 0) {
    int dev = 0, can = 0;
    cudaGetDevice(&dev);
    flush = (attr && attr(&can, 98 /*CU_DEVICE_ATTRIBUTE_CAN_FLUSH_REMOTE_WRITES*/, dev) == 0 && can) ? 1 : 0;
  }
  const unsigned flags = 0u /*CU_STREAM_WAIT_VALUE_GEQ*/ | (flush ? (1u << 30) /*CU_STREAM_WAIT_VALUE_FLUSH*/ : 0u);
  if (fn(stream, (unsigned long long)dev_ptr, value, flags) != 0)
    return fail(bt::ERR_CUDA, "cuStreamWaitValue32 failed");
  return 0;
}
int bt_ipc_open_handle(const void* handle, void** dev_ptr_out) {
  cudaIpcMemHandle_t h;
  memcpy(&h, handle, sizeof h);
  if (cudaIpcOpenMemHandle(dev_ptr_out, h, cudaIpcMemLazyEnablePeerAccess) != cudaSuccess)
    return cuda_fail("cudaIpcOpenMemHandle");
  return 0;
}
int bt_ipc_close(void* dev_ptr) {
  if (cudaIpcCloseMemHandle(dev_ptr) != cudaSuccess) return cuda_fail("cudaIpcCloseMemHandle");
  return 0;
}
int bt_enable_peer_access(int32_t peer_device) {
  cudaError_t e = cudaDeviceEnablePeerAccess(peer_device, 0);
  if (e == cudaErrorPeerAccessAlreadyEnabled) {
    cudaGetLastError();
    return 0;
  }
  if (e != cudaSuccess) return cuda_fail("cudaDeviceEnablePeerAccess");
  return 0;
}

// ------------------------------------------ C4 input / output layers (bt_embed.cu)
int bt_bert_tokens(uint64_t seed, int64_t step, const int64_t* step_dev, int32_t est_base, int32_t E, int32_t seqs,
                   int32_t vocab, int32_t npred, int32_t mask_id, int32_t* ids_dev, int32_t* mrow_dev,
                   int32_t* mlabel_dev, void* stream) {
  if (!ids_dev || !mrow_dev || !mlabel_dev) return fail(bt::ERR_INPUT, "null buffer");
  if (mask_id < 0 || mask_id >= vocab) return fail(bt::ERR_INPUT, "mask id %d outside the vocabulary", mask_id);
  return done(bt::emb_tokens_launch(seed, step, step_dev, est_base, E, seqs, vocab, npred, mask_id, ids_dev, mrow_dev,
                                    mlabel_dev, STREAM(stream)),
              "bt_bert_tokens");
}
int bt_bert_embed_fwd(const int32_t* ids_dev, const float* wemb_dev, const float* pemb_dev, int32_t T, int32_t D,
                      float* x32_dev, void* xb_dev, void* stream) {
  if (T < 1 || D < 4 || D % 8) return fail(bt::ERR_INPUT, "embedding %d x %d", T, D);
  return done(bt::emb_fwd_launch(ids_dev, wemb_dev, pemb_dev, T, D, x32_dev, xb_dev, STREAM(stream)),
              "bt_bert_embed_fwd");
}
int bt_rows_gather(const void* in_dev, const int32_t* rows_dev, int32_t R, int32_t D, void* out_dev, void* stream) {
  if (R < 1 || D % 8) return fail(bt::ERR_INPUT, "gather %d rows of %d", R, D);
  return done(bt::emb_gather_launch(in_dev, rows_dev, R, D, out_dev, STREAM(stream)), "bt_rows_gather");
}
int bt_rows_scatter(const void* src_dev, const int32_t* rows_dev, int32_t R, int32_t npred, int32_t T, int32_t D,
                    void* dst_dev, void* stream) {
  if (R < 1 || T < 1 || D % 8 || npred < 1) return fail(bt::ERR_INPUT, "scatter %d rows into %d", R, T);
  return done(bt::emb_scatter_launch(src_dev, rows_dev, R, npred, T, D, dst_dev, STREAM(stream)), "bt_rows_scatter");
}
int bt_bert_mlm_ce(const float* logits_dev, const int32_t* labels_dev, int32_t R, int32_t vocab, int32_t vocab_pad,
                   int32_t E, int32_t rows_per_est, void* dlogits_dev, float* row_loss_dev, float* loss_dev,
                   void* stream) {
  if (R < 1 || vocab < 2 || vocab > vocab_pad || R != E * rows_per_est)
    return fail(bt::ERR_INPUT, "cross-entropy over %d rows x %d classes (padded %d)", R, vocab, vocab_pad);
  return done(bt::emb_ce_launch(logits_dev, labels_dev, R, vocab, vocab_pad, E, rows_per_est, dlogits_dev, row_loss_dev,
                                loss_dev, STREAM(stream)),
              "bt_bert_mlm_ce");
}
int bt_bert_embed_grad_scratch(int32_t leaves, int32_t leaf_tokens, int32_t D, int64_t* ints_out,
                               int64_t* floats_out) {
  if (leaves < 1 || leaf_tokens < 128 || D < 8 || !ints_out || !floats_out) return fail(bt::ERR_INPUT, "bad shape");
  return bt::emb_grad_scratch(leaves, leaf_tokens, D, ints_out, floats_out);
}
int bt_bert_embed_grad(const void* dxa_dev, const float* dxb_dev, const int32_t* ids_dev, int32_t leaves,
                       int32_t leaf_tokens, int32_t D, int32_t* scratch_dev, float* partial_dev, float* dwemb_dev,
                       float* dpemb_dev, int64_t leaf_stride, void* stream) {
  if (leaves < 1 || leaf_tokens < 128 || leaf_tokens > 8192 || leaf_tokens % 128 || D % 8)
    return fail(bt::ERR_INPUT, "embedding gradient: %d leaves of %d tokens (<= 8192)", leaves, leaf_tokens);
  if (!scratch_dev || !partial_dev) return fail(bt::ERR_INPUT, "null scratch");
  return done(bt::emb_grad_launch(dxa_dev, dxb_dev, ids_dev, leaves, leaf_tokens, D, scratch_dev, partial_dev,
                                  dwemb_dev, dpemb_dev, leaf_stride, STREAM(stream)),
              "bt_bert_embed_grad");
}

// ------------------------------------------ per-EST BERT encoder step (C4)
static int bert_shape(int E, int Te, int D) {
  if (E < 1 || Te < 128 || Te % 128 || D % 256 || D > 1024)
    return fail(bt::ERR_INPUT, "bert shape E=%d Te=%d D=%d: need Te %% 128 == 0, D %% 256 == 0, D <= 1024", E, Te, D);
  return 0;
}
int bt_bert_data(uint64_t seed, int64_t step, int32_t est_base, int32_t E, int32_t Te, int32_t D, float* x32_dev,
                 void* xb_dev, float* target_dev, const int64_t* step_dev, void* stream) {
  if (int st = bert_shape(E, Te, D)) return st;
  if (!x32_dev || !xb_dev || !target_dev) return fail(bt::ERR_INPUT, "null pointer");
  return done(bt::bert_data_launch(seed, step, est_base, E, Te, D, x32_dev, xb_dev, target_dev, step_dev,
                                   STREAM(stream)),
              "bt_bert_data");
}
int bt_bert_attn_ex(int32_t backward, const void* qkv_dev, const void* dctx_dev, void* out_dev, int32_t E,
                    int32_t Te, int32_t D, int32_t heads, int32_t est_base, int32_t layers, int32_t layer, uint64_t seed,
                    int64_t step, float p, const int64_t* step_dev, float* stats_dev, void* stream) {
  return bt_bert_attn_ex2(backward, qkv_dev, dctx_dev, out_dev, E, Te, D, heads, est_base, layers, layer, seed, step, p,
                          step_dev, stats_dev, nullptr, stream);
}
int bt_bert_attn_ex2(int32_t backward, const void* qkv_dev, const void* dctx_dev, void* out_dev, int32_t E,
                     int32_t Te, int32_t D, int32_t heads, int32_t est_base, int32_t layers, int32_t layer, uint64_t seed,
                     int64_t step, float p, const int64_t* step_dev, float* stats_dev, uint32_t* mbits_dev,
                     void* stream) {
  if (int st = bert_shape(E, Te, D)) return st;
  if (((uintptr_t)mbits_dev) & 15) return fail(bt::ERR_INPUT, "attention keep bits must be 16-byte aligned");
  if (heads * 64 != D) return fail(bt::ERR_INPUT, "bert attention: head dim must be 64 (heads %d, D %d)", heads, D);
  if (!qkv_dev || !out_dev || (backward && !dctx_dev)) return fail(bt::ERR_INPUT, "null pointer");
  if (!(p >= 0.f && p < 1.f) || layer < 0 || layer >= layers) return fail(bt::ERR_CONFIG, "bad dropout / layer");
  return done(bt::bert_attn_launch(backward, qkv_dev, dctx_dev, out_dev, E * Te / 128, D, heads, Te / 128, est_base,
                                   layers, layer, seed, step, p, step_dev, STREAM(stream), stats_dev, mbits_dev),
              "bt_bert_attn");
}
int bt_bert_attn(int32_t backward, const void* qkv_dev, const void* dctx_dev, void* out_dev, int32_t E, int32_t Te,
                 int32_t D, int32_t heads, int32_t est_base, int32_t layers, int32_t layer, uint64_t seed, int64_t step,
                 float p, const int64_t* step_dev, void* stream) {
  return bt_bert_attn_ex(backward, qkv_dev, dctx_dev, out_dev, E, Te, D, heads, est_base, layers, layer, seed, step, p,
                         step_dev, nullptr, stream);
}
int bt_bert_ln_fwd(const float* resid_dev, const void* branch_dev, const float* bias_dev, const float* gamma_dev,
                   const float* beta_dev, float* xsum_dev, float* stats_dev, float* y32_dev, void* yb_dev, int32_t E,
                   int32_t Te, int32_t D, int32_t est_base, int32_t layers, int32_t layer, int32_t site, uint64_t seed,
                   int64_t step, float p, float eps, const int64_t* step_dev, void* stream) {
  if (int st = bert_shape(E, Te, D)) return st;
  if (!resid_dev || !branch_dev || !bias_dev || !gamma_dev || !beta_dev || !xsum_dev || !stats_dev || !yb_dev)
    return fail(bt::ERR_INPUT, "null pointer");
  if (!(p >= 0.f && p < 1.f) || (site != 0 && site != 1)) return fail(bt::ERR_CONFIG, "bad dropout / site");
  return done(bt::bert_ln_launch(0, resid_dev, branch_dev, bias_dev, gamma_dev, beta_dev, xsum_dev, stats_dev, y32_dev,
                                 yb_dev, nullptr, E, Te, D, est_base, layers, layer, site, seed, step, p, eps,
                                 step_dev, STREAM(stream)),
              "bt_bert_ln_fwd");
}
int bt_bert_ln_fwd_rc(const float* prev_xsum_dev, const float* prev_stats_dev, const float* prev_gamma_dev,
                      const float* prev_beta_dev, const void* branch_dev, const float* bias_dev, const float* gamma_dev,
                      const float* beta_dev, float* xsum_dev, float* stats_dev, float* y32_dev, void* yb_dev, int32_t E,
                      int32_t Te, int32_t D, int32_t est_base, int32_t layers, int32_t layer, int32_t site,
                      uint64_t seed, int64_t step, float p, float eps, const int64_t* step_dev, void* stream) {
  if (int st = bert_shape(E, Te, D)) return st;
  if (!prev_xsum_dev || !prev_stats_dev || !prev_gamma_dev || !prev_beta_dev || !branch_dev || !bias_dev ||
      !gamma_dev || !beta_dev || !xsum_dev || !stats_dev || !yb_dev)
    return fail(bt::ERR_INPUT, "null pointer");
  if (!(p >= 0.f && p < 1.f) || (site != 0 && site != 1)) return fail(bt::ERR_CONFIG, "bad dropout / site");
  return done(bt::bert_ln_launch(0, nullptr, branch_dev, bias_dev, gamma_dev, beta_dev, xsum_dev, stats_dev, y32_dev,
                                 yb_dev, nullptr, E, Te, D, est_base, layers, layer, site, seed, step, p, eps,
                                 step_dev, STREAM(stream), prev_xsum_dev, prev_stats_dev, prev_gamma_dev,
                                 prev_beta_dev),
              "bt_bert_ln_fwd_rc");
}
int bt_bert_ln_bwd(const void* dy1_dev, const float* dy2_dev, const float* xsum_dev, const float* stats_dev,
                   const float* gamma_dev, float* dx_dev, void* dbranch_dev, float* part_dev, int32_t E, int32_t Te,
                   int32_t D, int32_t est_base, int32_t layers, int32_t layer, int32_t site, uint64_t seed,
                   int64_t step, float p, const int64_t* step_dev, void* stream) {
  if (int st = bert_shape(E, Te, D)) return st;
  if (!dy1_dev || !xsum_dev || !stats_dev || !gamma_dev || !dx_dev || !dbranch_dev || !part_dev)
    return fail(bt::ERR_INPUT, "null pointer");
  if (!(p >= 0.f && p < 1.f) || (site != 0 && site != 1)) return fail(bt::ERR_CONFIG, "bad dropout / site");
  return done(bt::bert_ln_launch(1, dy2_dev, dy1_dev, nullptr, gamma_dev, nullptr, (float*)xsum_dev,
                                 (float*)stats_dev, dx_dev, dbranch_dev, part_dev, E, Te, D, est_base, layers, layer,
                                 site, seed, step, p, 0.f, step_dev, STREAM(stream)),
              "bt_bert_ln_bwd");
}
int bt_bert_ln_fold(const float* part_dev, int32_t E, int32_t Te, int32_t D, float* dgamma_dev, float* dbeta_dev,
                    float* dbias_dev, int64_t est_stride, void* stream) {
  if (int st = bert_shape(E, Te, D)) return st;
  if (!part_dev || !dgamma_dev || !dbeta_dev || !dbias_dev) return fail(bt::ERR_INPUT, "null pointer");
  return done(bt::bert_ln_fold_launch(part_dev, E, Te, D, dgamma_dev, dbeta_dev, dbias_dev, est_stride,
                                      STREAM(stream)),
              "bt_bert_ln_fold");
}
int bt_bert_mse(const float* y_dev, const float* target_dev, int32_t E, int32_t Te, int32_t D, void* dy_dev,
                float* partials_dev, float* loss_dev, void* stream) {
  if (int st = bert_shape(E, Te, D)) return st;
  if (!y_dev || !target_dev || !dy_dev || !partials_dev || !loss_dev) return fail(bt::ERR_INPUT, "null pointer");
  return done(bt::bert_mse_launch(y_dev, target_dev, E, Te, D, dy_dev, partials_dev, loss_dev, STREAM(stream)),
              "bt_bert_mse");
}
int bt_colsum_fold(const float* part_dev, int32_t E, int32_t chunks, int32_t C, float* out_dev, int64_t out_stride,
                   void* stream) {
  if (!part_dev || !out_dev) return fail(bt::ERR_INPUT, "null pointer");
  if (E < 1 || chunks < 1 || C < 1 || out_stride < C) return fail(bt::ERR_INPUT, "colsum fold shape");
  return done(bt::colsum_fold_launch(part_dev, E, chunks, C, out_dev, out_stride, STREAM(stream)), "bt_colsum_fold");
}
int bt_colsum_bf16_strided(const void* in_dev, int32_t E, int32_t R, int32_t C, float* out_dev, int64_t out_stride,
                           float* scratch_dev, void* stream) {
  if (E < 1 || R < 1 || C < 1 || C % 8 || out_stride < C) return fail(bt::ERR_INPUT, "colsum shape");
  if (!in_dev || !out_dev) return fail(bt::ERR_INPUT, "null pointer");
  return done(bt::colsum_bf16_strided_launch(in_dev, E, R, C, out_dev, out_stride, scratch_dev, STREAM(stream)),
              "bt_colsum_bf16_strided");
}
int bt_cast_weights_bf16(const float* const* w_dev, void* const* wb_dev, void* const* wt_dev, const int32_t* rows,
                         const int32_t* cols, int32_t n, void* stream) {
  if (n < 1 || n > 64) return fail(bt::ERR_INPUT, "cast table of %d matrices (1..64)", n);
  return done(bt::bert_cast_weights_launch(w_dev, wb_dev, wt_dev, rows, cols, n, STREAM(stream)),
              "bt_cast_weights_bf16");
}

// ------------------------------------ per-EST ResNet-18 step with BatchNorm (C3)
int bt_cnn_data(uint64_t seed, const int64_t* cursor_dev, int32_t est_base, int32_t E, int32_t B, void* x_dev,
                int32_t* labels_dev, void* stream) {
  if (E < 1 || B < 1 || !cursor_dev || !x_dev || !labels_dev) return fail(bt::ERR_INPUT, "bt_cnn_data arguments");
  return done(bt::cnn_data_launch(seed, cursor_dev, est_base, E, B, x_dev, labels_dev, STREAM(stream)), "bt_cnn_data");
}
int bt_cnn_im2col(const void* src_dev, void* col_dev, int32_t N, int32_t Hs, int32_t Ws, int32_t C, int32_t Ho,
                  int32_t Wo, int32_t KH, int32_t KW, int32_t stride, int32_t pad, int32_t transposed, void* stream) {
  if (!src_dev || !col_dev || N < 1 || C % 8 || C < 8 || stride < 1 || KH < 1 || KW < 1 || Ho < 1 || Wo < 1)
    return fail(bt::ERR_INPUT, "bt_cnn_im2col shape (C %% 8 == 0)");
  return done(bt::cnn_im2col_launch(src_dev, col_dev, N, Hs, Ws, C, Ho, Wo, KH, KW, stride, pad, transposed,
                                    STREAM(stream)),
              "bt_cnn_im2col");
}
int bt_cnn_bn_stats(int32_t mode, const void* z_dev, const void* dy_dev, const void* y_dev, float* mean_dev,
                    float* rstd_dev, float* sg_dev, float* sgx_dev, float* part_dev, float* run_mean_dev,
                    float* run_var_dev, int64_t run_stride, float* dgamma_dev, float* dbeta_dev, int64_t grad_stride,
                    int32_t E, int32_t R, int32_t C, float eps, void* stream) {
  if ((mode != 0 && mode != 2) || E < 1 || R < 2 || !(C == 8 || C == 16 || C == 32 || C % 64 == 0) || C > 2048 ||
      !z_dev || !mean_dev || !part_dev)
    return fail(bt::ERR_INPUT, "bt_cnn_bn_stats arguments (mode 0 or 2; C in {8, 16, 32} or a multiple of 64)");
  if (mode == 0 && (!rstd_dev || !run_mean_dev || !run_var_dev)) return fail(bt::ERR_INPUT, "mode 0 needs rstd/run");
  if (mode == 2 && (!dy_dev || !y_dev || !rstd_dev || !sg_dev || !sgx_dev || !dgamma_dev || !dbeta_dev))
    return fail(bt::ERR_INPUT, "mode 2 needs dy, y, rstd, sums and gradient slots");
  return done(bt::cnn_bn_stats_launch(mode, z_dev, dy_dev, y_dev, mean_dev, rstd_dev, sg_dev, sgx_dev, part_dev,
                                      run_mean_dev, run_var_dev, run_stride, dgamma_dev, dbeta_dev, grad_stride, E, R,
                                      C, eps, STREAM(stream)),
              "bt_cnn_bn_stats");
}
int bt_cnn_bn_apply(const void* z_dev, const void* res_dev, const float* mean_dev, const float* rstd_dev,
                    const float* gamma_dev, const float* beta_dev, int32_t E, int32_t R, int32_t C, int32_t relu,
                    void* y_dev, void* stream) {
  if (E < 1 || R < 1 || C % 8 || !z_dev || !y_dev || !mean_dev || !rstd_dev || !gamma_dev || !beta_dev ||
      (((uintptr_t)mean_dev | (uintptr_t)rstd_dev | (uintptr_t)gamma_dev | (uintptr_t)beta_dev) & 15))
    return fail(bt::ERR_INPUT, "bt_cnn_bn_apply arguments (per-channel vectors 16-byte aligned)");
  return done(bt::cnn_bn_apply_launch(z_dev, res_dev, mean_dev, rstd_dev, gamma_dev, beta_dev, E, R, C, relu, y_dev,
                                      STREAM(stream)),
              "bt_cnn_bn_apply");
}
int bt_cnn_bn_bwd(const void* z_dev, const void* dy_dev, const void* y_dev, const float* mean_dev,
                  const float* rstd_dev, const float* sg_dev, const float* sgx_dev, const float* gamma_dev, int32_t E,
                  int32_t R, int32_t C, void* dz_dev, void* stream) {
  if (E < 1 || R < 1 || C % 8 || !z_dev || !dy_dev || !y_dev || !dz_dev || !mean_dev || !rstd_dev || !sg_dev ||
      !sgx_dev || !gamma_dev ||
      (((uintptr_t)mean_dev | (uintptr_t)rstd_dev | (uintptr_t)sg_dev | (uintptr_t)sgx_dev | (uintptr_t)gamma_dev) & 15))
    return fail(bt::ERR_INPUT, "bt_cnn_bn_bwd arguments (per-channel vectors 16-byte aligned)");
  return done(bt::cnn_bn_bwd_launch(z_dev, dy_dev, y_dev, mean_dev, rstd_dev, sg_dev, sgx_dev, gamma_dev, E, R, C,
                                    dz_dev, STREAM(stream)),
              "bt_cnn_bn_bwd");
}
int bt_cnn_add(const void* a_dev, const void* b_dev, const void* y_dev, int64_t n, void* out_dev, void* stream) {
  if (!a_dev || !b_dev || !out_dev || n % 8) return fail(bt::ERR_INPUT, "bt_cnn_add arguments");
  return done(bt::cnn_add_launch(a_dev, b_dev, y_dev, n, out_dev, STREAM(stream)), "bt_cnn_add");
}
int bt_cnn_upsample(const void* src_dev, int64_t N, int32_t Hs, int32_t Ws, int32_t C, int32_t s, void* up_dev,
                    void* stream) {
  if (!src_dev || !up_dev || N < 1 || Hs < 1 || Ws < 1) return fail(bt::ERR_INPUT, "bt_cnn_upsample arguments");
  return done(bt::cnn_upsample_launch(src_dev, N, Hs, Ws, C, s, up_dev, STREAM(stream)),
              "bt_cnn_upsample (C a power of two >= 8, s in {1, 2})");
}
int bt_cnn_filter_taps(const float* const* w_dev, void* const* out_dev, const int32_t* co, const int32_t* taps,
                       const int32_t* ci, const int32_t* class_taps, const int32_t* tap_map, int32_t n, void* stream) {
  if (!w_dev || !out_dev || !co || !taps || !ci || !class_taps || !tap_map || n < 1 || n > 16)
    return fail(bt::ERR_INPUT, "bt_cnn_filter_taps arguments (1 <= n <= 16)");
  return done(bt::cnn_filter_taps_launch(w_dev, out_dev, co, taps, ci, class_taps, tap_map, n, STREAM(stream)),
              "bt_cnn_filter_taps (1 <= class taps <= 9, map entries < taps)");
}
int bt_cnn_add_s2(const void* const* a_dev, const void* const* b_dev, void* out_dev, int64_t N, int32_t Hs, int32_t Ws,
                  int32_t C, void* stream) {
  if (!out_dev || N < 1 || Hs < 1 || Ws < 1) return fail(bt::ERR_INPUT, "bt_cnn_add_s2 arguments");
  return done(bt::cnn_add_s2_launch(a_dev, b_dev, out_dev, N, Hs, Ws, C, STREAM(stream)),
              "bt_cnn_add_s2 (C a power of two >= 8)");
}
int bt_cnn_head(const void* x_dev, const int32_t* labels_dev, const float* w_dev, const float* b_dev, int32_t E,
                int32_t B, float* dw_dev, float* db_dev, int64_t grad_stride, float* loss_dev, void* dx_dev,
                void* stream) {
  if (E < 1 || B < 1 || B > 96 || !x_dev || !labels_dev || !w_dev || !b_dev || !dw_dev || !db_dev || !loss_dev ||
      !dx_dev)
    return fail(bt::ERR_INPUT, "bt_cnn_head arguments (B <= 96)");
  return done(bt::cnn_head_launch(x_dev, labels_dev, w_dev, b_dev, E, B, dw_dev, db_dev, grad_stride, loss_dev, dx_dev,
                                  STREAM(stream)),
              "bt_cnn_head");
}
int bt_fold_splits(const float* part_dev, int32_t E, int32_t splits, int64_t n, float* out_dev, int64_t out_stride,
                   void* stream) {
  if (!part_dev || !out_dev || E < 1 || splits < 1 || n < 4 || n % 4 || out_stride < n || out_stride % 4)
    return fail(bt::ERR_INPUT, "bt_fold_splits arguments");
  return done(bt::cnn_fold_splits_launch(part_dev, E, splits, n, out_dev, out_stride, STREAM(stream)),
              "bt_fold_splits");
}
int bt_cnn_conv_weights(const float* const* w_dev, void* const* wb_dev, void* const* wt_dev, const int32_t* co,
                        const int32_t* taps, const int32_t* ci, const int32_t* flip, int32_t n, void* stream) {
  if (n < 1 || n > 32) return fail(bt::ERR_INPUT, "conv weight table of %d (1..32)", n);
  return done(bt::cnn_conv_weights_launch(w_dev, wb_dev, wt_dev, co, taps, ci, flip, n, STREAM(stream)),
              "bt_cnn_conv_weights");
}

}  // extern "C"
