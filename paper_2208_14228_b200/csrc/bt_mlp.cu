// bt_mlp.cu -- fused, persistent data-parallel step for the reference MLP.
//
// One launch runs K mini-batches of engine.run_minibatch (engine.py:271-329):
//   B  rows (device sampler: epoch lists + counter-form worker-RNG jitter,
//      sampling.py:160-172, or an explicit split_by_rank global batch,
//      engine.py:261-268) -> hidden layer + tanh + dropout (model.py:141-163);
//   C  output error, upstream factor gy, dz, tracked-stat row means
//      (model.py:165-179, 194) -- fused into B: a row's 16 lanes sit in one warp;
//   E  161 per-EST gradients, each a batch-dim reduce_sum in the EST's
//      executor variant (model.py:183-192) -> EST gradient slot; per-EST loss,
//      TrackedStat update and dropout-RNG advance (model.py:173, 99-104);
//   F  the fixed-order allreduce in executor 0's variant (buckets.py:115-123,
//      keyed by EST rank, never by GPU/CTA) fused with /E and momentum SGD
//      (model.py:206-212).
// Layout: CTA c owns ESTs [c*epc, (c+1)*epc).  Everything a step touches is
// staged in shared memory for the whole launch (parameters, velocity, EST
// RNG/stat slots, the rotation table, the EST gradient slots, and -- when they
// fit -- the dataset and this launch's index lists).
// Exchange: on a thread-block cluster every CTA pushes its EST slots into
// every CTA's step-parity slot array with st.async (DSMEM store + mbarrier
// complete_tx); a CTA waits on its own mbarrier for all E_total*P*8 bytes, so
// there is no cluster-wide barrier and no release fence per step.  Stage F is
// computed by EVERY CTA redundantly (bit-identical: same inputs, same order).
// Parameters/velocity are double-buffered so a step commits with one CTA
// barrier (and only when every synchronized gradient is finite).
// Every binary64 op is an explicit _rn intrinsic (no FMA contraction) and tanh
// is glibc's (bt_libm.cuh): results are bit-identical to the reference.
#include "bt_common.cuh"
#include "bt_libm.cuh"
#include "bt_mlp.cuh"

namespace bt {

constexpr int MLP_THREADS = 512;
constexpr int BT_MAX_FUSED_E = 256;  // ESTs of one fused step
constexpr int MAX_CLUSTER_CTAS = 8;  // portable thread-block cluster size
constexpr int PAD_P = 168;  // 161 rounded up to a multiple of 8 doubles
constexpr int FOLD_LEVELS = 10;  // trees of up to 2^9 = 512 leaves

__device__ __forceinline__ uint32_t ld_acquire_u32(const uint32_t* p) {
  uint32_t v;
  asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}

// Software grid barrier (all CTAs co-resident: cooperative launch).  Bounded
// spin: a barrier that never completes reports ERR_CUDA instead of hanging.
__device__ __forceinline__ bool grid_sync(uint32_t* bar, uint32_t target, int32_t* flags) {
  __shared__ int s_ok;
  __syncthreads();
  if (threadIdx.x == 0) {
    __threadfence();
    atomicAdd(bar, 1u);
    long long t0 = clock64();
    int ok = 1;
    while (ld_acquire_u32(bar) < target) {
      if (clock64() - t0 > (1ll << 36)) {  // ~30 s at 2 GHz
        atomicCAS(flags + FLAG_STATUS, 0, (int)ERR_CUDA);
        ok = 0;
        break;
      }
    }
    __threadfence();
    s_ok = ok;
  }
  __syncthreads();
  return s_ok != 0;
}

// reduce_sum over the B rows of one EST in its executor's variant.  FB >= 0:
// every EST's variant is known at compile time; otherwise `fan` (run time).
template <int BT, int FB, class Gen>
__device__ __forceinline__ double fold_rows(int nb, int fan, Gen gen) {
  if constexpr (BT > 0) {
    double v[BT];
#pragma unroll
    for (int r = 0; r < BT; ++r) v[r] = gen(r);
    if constexpr (FB >= 0) {
      return TreeLevel<BT, FB>::run(v);
    } else {
      if (fan == 0 || fan >= BT) return TreeLevel<BT, 0>::run(v);  // Tree(f >= n) folds like Sequential
      if (fan == 2) return TreeLevel<BT, 2>::run(v);
      StreamFold<double, FOLD_LEVELS> f;
      f.init(fan);
#pragma unroll
      for (int r = 0; r < BT; ++r) f.push(v[r]);
      return f.finish();
    }
  } else {
    StreamFold<double, FOLD_LEVELS> f;
    f.init(fan);
    for (int r = 0; r < nb; ++r) f.push(gen(r));
    return f.finish();
  }
}

// The allreduce fold of one parameter over N EST slots (slot of leaf k is
// (start+k) mod N), register-resident with a compile-time tree shape F.
// `ld(q)` returns EST slot q's value.
template <int N, int F, class Ld>
__device__ __forceinline__ double fold_ranks_t(int start, Ld ld) {
  double v[N];
#pragma unroll
  for (int k = 0; k < N; ++k) {
    int q = start + k;
    q -= q >= N ? N : 0;
    v[k] = ld(q);
  }
  return TreeLevel<N, F>::run(v);
}

template <int N, class Ld>
__device__ __forceinline__ double fold_ranks_n(int fan, int start, Ld ld) {  // fan in {0, 2}
  return fan == 0 ? fold_ranks_t<N, 0>(start, ld) : fold_ranks_t<N, 2>(start, ld);
}

// Register tree for the common shapes (power-of-two E, Sequential / Tree(2));
// everything else takes the (compact) register StreamFold.
template <class Ld>
__device__ __forceinline__ bool fold_ranks_ct(int n, int fan, int start, Ld ld, double* out) {
  if (!(fan == 0 || fan == 2)) return false;
  switch (n) {
    case 1: *out = ld(0); return true;
    case 2: *out = fold_ranks_n<2>(fan, start, ld); return true;
    case 4: *out = fold_ranks_n<4>(fan, start, ld); return true;
    case 8: *out = fold_ranks_n<8>(fan, start, ld); return true;
    case 16: *out = fold_ranks_n<16>(fan, start, ld); return true;
    case 32: *out = fold_ranks_n<32>(fan, start, ld); return true;
    case 64: *out = fold_ranks_n<64>(fan, start, ld); return true;
    default: return false;
  }
}

// Any (E, fanin): the register StreamFold over the rotated slot order.
template <class Ld>
__device__ __forceinline__ double fold_ranks_any(int n, int fan, int start, Ld ld) {
  double out;
  if (fold_ranks_ct(n, fan, start, ld, &out)) return out;
  StreamFold<double, 12> f;
  f.init(fan);
  for (int k = 0; k < n; ++k) {
    int q = start + k;
    q -= q >= n ? n : 0;
    f.push(ld(q));
  }
  return f.finish();
}

struct MlpHostSignal {  // bt_mlp_run's request: results to mapped host memory + a done word (see MlpLaunch)
  double* out;
  uint32_t* done;
  uint32_t seq;
};
struct MlpLaunch {  // launcher-computed shared-memory plan
  int stage_data;   // dataset copied into shared memory
  int stage_idx;    // this launch's index lists copied into shared memory
  int grads_smem;   // EST gradient slots [E_total][P] in shared memory (fused, non-cluster mode)
  int cluster;      // fused mode on a thread-block cluster: slots pushed through DSMEM
  unsigned long long* timing;  // optional [9] per-stage clock64 sums (bt_mlp_step_profiled)
  // Host signal (single-device compact build): the epilogue copies the K x E_total losses and the 4 status
  // words into mapped pinned host memory and then writes done_seq to host_done (system-scope release), so
  // the host sees the results without a device-to-host copy and a stream synchronisation.
  double* host_out;
  uint32_t* host_done;
  uint32_t done_seq;
};

// ---- cluster plumbing (PTX) -------------------------------------------------
__device__ __forceinline__ void cluster_barrier() {  // all threads of all CTAs; release/acquire
  asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}
__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
// shared::cluster window address of this CTA's shared address `local` in CTA `rank`
__device__ __forceinline__ uint32_t cluster_map32(uint32_t local, int rank) {
  uint32_t out;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(out) : "r"(local), "r"(rank));
  return out;
}
__device__ __forceinline__ void mbar_init(uint32_t bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(bar), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_init_fence() {  // make mbarrier.init visible to cluster peers
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}
__device__ __forceinline__ void mbar_arrive_expect_tx(uint32_t bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bar), "r"(bytes) : "memory");
}
__device__ __forceinline__ double ld_shared_f64(uint32_t addr) {
  double v;
  asm volatile("ld.shared.f64 %0, [%1];" : "=d"(v) : "r"(addr) : "memory");
  return v;
}
__device__ __forceinline__ void st_shared_f64(uint32_t addr, double v) {
  asm volatile("st.shared.f64 [%0], %1;" ::"r"(addr), "d"(v) : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint32_t bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(bar) : "memory");
}
__device__ __forceinline__ bool mbar_try_wait(uint32_t bar, uint32_t parity) {
  uint32_t ok;
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\t"
      "selp.u32 %0, 1, 0, p;\n\t}"
      : "=r"(ok)
      : "r"(bar), "r"(parity)
      : "memory");
  return ok != 0;
}
__device__ __forceinline__ void cluster_arrive() {
  asm volatile("barrier.cluster.arrive.release.aligned;" ::: "memory");
}
__device__ __forceinline__ void cluster_wait() {
  asm volatile("barrier.cluster.wait.acquire.aligned;" ::: "memory");
}
// Bulk copy global -> this CTA's shared memory, counted on its mbarrier (16-byte aligned sizes).
__device__ __forceinline__ void bulk_g2s(uint32_t dst, const void* src, uint32_t bytes, uint32_t bar) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(dst),
               "l"(src), "r"(bytes), "r"(bar)
               : "memory");
}
// Bulk copy global -> the same shared offset in every CTA of `mask`, counted on each CTA's mbarrier
// (the same offset too).  bytes and both addresses 16-byte aligned.
__device__ __forceinline__ void bulk_multicast(uint32_t dst, const void* src, uint32_t bytes, uint32_t bar,
                                               uint16_t mask) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.multicast::cluster [%0], [%1], %2, [%3], %4;" ::
          "r"(dst),
      "l"(src), "r"(bytes), "r"(bar), "h"(mask)
      : "memory");
}
// DSMEM store into a cluster peer that also counts 8 bytes on the peer's mbarrier
__device__ __forceinline__ void st_async_f64(uint32_t addr, double v, uint32_t remote_bar) {
  asm volatile("st.async.shared::cluster.mbarrier::complete_tx::bytes.f64 [%0], %1, [%2];" ::"r"(addr), "d"(v),
               "r"(remote_bar)
               : "memory");
}

// Per-stage cycle accounting for profiling builds of a launch (thread 0's view
// of each barrier); compiled in, branch-predicated off when L.timing is null.
#define BT_TICK(k)                                     \
  if (L.timing && tid == 0) {                          \
    const long long now_ = clock64();                  \
    tacc[k] += (unsigned long long)(now_ - tlast);     \
    tlast = now_;                                      \
  }

// Generic build: BT = compile-time rows per EST (0 = run time); any E_total,
// per-EST variants, explicit or sampled rows, cluster / grid / single-CTA.
// (mlp_step_spec_kernel below is the compact build for the common shapes.)
template <int BT>
__global__ void __launch_bounds__(MLP_THREADS) mlp_step_kernel(const __grid_constant__ bt_mlp_args a,
                                                               const MlpLaunch L) {
  constexpr bool SPEC = false;
  constexpr int ET = 0, FB = -1, FC = -1;
  extern __shared__ __align__(16) double sm[];
  const int tid = threadIdx.x, T = blockDim.x;  // T >= BT_P (launcher): thread p owns parameter p in stage F
  const int cta = blockIdx.x, G = gridDim.x;
  const int nb = BT > 0 ? BT : a.B;
  const int epc = a.est_per_cta;
  const int e0 = cta * epc;
  const int ne = min(epc, a.E - e0);
  const int nrows = ne * nb;
  const int rows_cap = epc * nb;
  const int Et = SPEC ? ET : a.E_total;
  const bool staged = SPEC || (L.stage_idx && L.stage_data);

  double* s_par = sm;                            // current parameters / velocity ...
  double* s_vel = s_par + PAD_P;
  double* s_par_n = s_vel + PAD_P;               // ... and the next step's (double buffer)
  double* s_vel_n = s_par_n + PAD_P;
  double* s_x = s_vel_n + PAD_P;                 // [rows][8] jittered inputs
  double* s_y = s_x + rows_cap * BT_INPUT_DIM;   // [rows]
  double* s_act = s_y + rows_cap;                // [rows][16] tanh outputs
  double* s_msk = s_act + rows_cap * BT_HIDDEN;  // [rows][16] dropout masks
  double* s_hid = s_msk + rows_cap * BT_HIDDEN;  // [rows][16] acts*mask
  double* s_dz = s_hid + rows_cap * BT_HIDDEN;   // [rows][16]
  double* s_gy = s_dz + rows_cap * BT_HIDDEN;    // [rows]
  double* s_e2 = s_gy + rows_cap;                // [rows]
  double* s_rm = s_e2 + rows_cap;                // [rows] row means of acts
  double* s_mean = s_rm + rows_cap;              // [epc]
  uint64_t* s_rng = (uint64_t*)(s_mean + epc);   // [epc]
  uint64_t* s_cnt = s_rng + epc;                 // [epc]
  double* s_grad = (double*)(s_cnt + epc);  // [E_total][P] when L.grads_smem; [2][E_total][P] when L.cluster
  double* s_data = s_grad + (L.cluster ? (size_t)2 * Et * BT_P : (L.grads_smem ? (size_t)Et * BT_P : 0));
  double* s_jit = s_data + (L.stage_data ? (size_t)a.dataset_rows * BT_ROW : 0);  // [K][epc][B] when L.stage_idx
  int32_t* s_rot = (int32_t*)(s_jit + (L.stage_idx ? (size_t)a.K * rows_cap : 0));  // [P]
  int32_t* s_fan = s_rot + PAD_P;                // [epc] batch-reduction fanin per local EST
  int32_t* s_idx = s_fan + ((epc + 1) & ~1);     // [K][epc][B] when L.stage_idx

  __shared__ uint32_t s_peer[MAX_CLUSTER_CTAS];     // cluster: CTA r's slot array (shared::cluster)
  __shared__ uint32_t s_peerbar[MAX_CLUSTER_CTAS];  // cluster: CTA r's mbarrier pair
  __shared__ __align__(8) uint64_t s_mbar[2];       // cluster: "all slots of step parity q arrived"

  if (a.flags[FLAG_STATUS] != 0) return;  // sticky error from an earlier launch (same for every CTA)
  if (L.cluster) {
    if (tid == 0) {
      mbar_init(smem_u32(&s_mbar[0]), 1);
      mbar_init(smem_u32(&s_mbar[1]), 1);
      mbar_init_fence();
    }
    for (int r = tid; r < G; r += T) {
      s_peer[r] = cluster_map32(smem_u32(s_grad), r);
      s_peerbar[r] = cluster_map32(smem_u32(&s_mbar[0]), r);
    }
  }

  // ---- launch prologue: stage state in shared memory -----------------------
  const double* rep0 = a.replicas;
  int bad = 0;
  for (int i = tid; i < BT_P; i += T) {
    const double p0 = rep0[i];
    const double v0 = a.fuse_reduce ? rep0[BT_P + i] : 0.0;  // grads-only seam passes bare params
    s_par[i] = p0;
    s_vel[i] = v0;
    s_rot[i] = a.rot ? a.rot[i] : 0;
    for (int x = 1; x < a.X; ++x) {  // replica agreement, bytewise (engine.py:246-258)
      const double* rx = a.replicas + (size_t)x * 2 * BT_P;
      bad |= d2u(rx[i]) != d2u(p0);
      if (a.fuse_reduce) bad |= d2u(rx[BT_P + i]) != d2u(v0);
    }
  }
  int hint_bad = 0;
  for (int el = tid; el < ne; el += T) {
    s_rng[el] = a.rng[e0 + el];
    s_mean[el] = a.stat_mean[e0 + el];
    s_cnt[el] = a.stat_count[e0 + el];
    s_fan[el] = a.est_fanin[e0 + el];
    if (SPEC) hint_bad |= s_fan[el] != FB;
  }
  if (L.stage_data) {
    const int64_t nd = a.dataset_rows * BT_ROW;
    for (int64_t i = tid; i < nd; i += T) s_data[i] = a.dataset[i];
  }
  if (L.stage_idx) {
    for (int it = tid; it < a.K * ne * nb; it += T) {
      const int s = it / (ne * nb), rem = it - s * ne * nb;
      const int el = rem / nb, r = rem - el * nb;
      const int64_t gstep = a.step0 + s, epoch = gstep / a.spe, local = gstep % a.spe;
      const int eg = a.est_base + e0 + el;
      const int32_t* lst = a.lists + ((size_t)(epoch - a.epoch_base) * Et + eg) * (size_t)(a.spe * nb);
      const int q = (s * epc + el) * nb + r;
      s_idx[q] = lst[local * nb + r];
      double ju = 0.0;
      if (a.jitter != 0.0) {  // one uniform per row of worker_rng(seed, epoch, local, est) (sampling.py:99-170)
        const uint64_t w = derive5(TAG_DATA_WORKER, a.seed, (uint64_t)epoch, (uint64_t)local, (uint64_t)eg);
        ju = dmul(dsub(unit_float(draw_raw(w, (uint64_t)r)), 0.5), a.jitter);
      }
      s_jit[q] = ju;
    }
  }
  // every CTA reads the same replicas / fanins, so all CTAs take the same exit
  const int prologue = __syncthreads_or(bad | (hint_bad << 1));
  if (prologue) {
    if (cta == 0 && tid == 0) {
      a.flags[FLAG_STATUS] = (prologue & 1) ? ERR_CORRUPTION : ERR_INPUT;
      a.flags[FLAG_STEP] = 0;
    }
    return;
  }
  if (L.cluster) cluster_barrier();  // every peer's mbarriers are initialised before the first push

  const double rate = a.rate;
  const double keep = rate >= 1.0 ? 0.0 : ddiv(1.0, dsub(1.0, rate));  // model.py:150
  // true divisions of the reference (model.py:173,176,194, buckets.py:123); exact multiplies for powers of two
  const IntDivisor divB = IntDivisor::of(nb), divH = IntDivisor::of(BT_HIDDEN), divE = IntDivisor::of(Et);
  const double* data = L.stage_data ? s_data : a.dataset;
  const bool jit = !a.rows && a.jitter != 0.0;
  const uint32_t slot_bytes = (uint32_t)Et * BT_P * (uint32_t)sizeof(double);  // one step's arrivals per CTA
  uint32_t phases = 0;  // cluster: bit q = parity of the next completion of s_mbar[q]
  int s = 0;
  int64_t epoch = a.rows ? 0 : a.step0 / a.spe, local = a.rows ? 0 : a.step0 % a.spe;

  unsigned long long tacc[9] = {0, 0, 0, 0, 0, 0, 0, 0, 0};
  long long tlast = clock64();
  for (; s < a.K; ++s) {
    const int64_t gstep = a.step0 + s;
    const int par = (int)(gstep & 1);
    if (s > 0 && !a.rows && ++local == a.spe) {  // incremental (no 64-bit division per step)
      local = 0;
      ++epoch;
    }

    // ---- B+C: one 16-lane group per row (lane j = hidden unit j) ----------
    // B: row gather + jitter, pre-activation, tanh, dropout (model.py:141-163).
    // C: every lane of the group reads the row's 16 products w2[j]*h[j] and 16
    // activations (shared-memory broadcast) and runs the two sequential
    // 16-term folds (output and row mean, model.py:168-171, 194) -- identical
    // bits on every lane -- then lane j writes dz[r][j] = ((gy*w2[j])*mask)*(1-a*a)
    // (model.py:179).  A row's lanes share a warp, so B -> C is a __syncwarp.
    {
      const int span = ((nrows * BT_HIDDEN + 31) / 32) * 32;
#pragma unroll 1
      for (int it = tid; it < span; it += T) {
        const bool valid = it < nrows * BT_HIDDEN;
        const int row = valid ? it >> 4 : 0, j = it & 15;
        const int el = row / nb, r = row - el * nb;
        const int eg = a.est_base + e0 + el;  // global virtual rank
        double x[BT_ROW];  // 8 inputs, then y
        double ju = 0.0;
        if (staged) {  // the common path: shared-memory rows (LDS), staged index + jitter
          const int q = (s * epc + el) * nb + r;
          const double* srcs = s_data + (size_t)s_idx[q] * BT_ROW;
          ju = s_jit[q];
#pragma unroll
          for (int i = 0; i < BT_ROW; ++i) x[i] = srcs[i];
        } else {
          const double* src;
          if (a.rows) {  // split_by_rank: row r of rank k is global row r*E+k
            src = a.rows + ((size_t)s * nb * Et + (size_t)r * Et + eg) * BT_ROW;
          } else if (L.stage_idx) {
            const int q = (s * epc + el) * nb + r;
            src = data + (size_t)s_idx[q] * BT_ROW;
            ju = s_jit[q];
          } else {
            const int32_t* lst = a.lists + ((size_t)(epoch - a.epoch_base) * Et + eg) * (size_t)(a.spe * nb);
            src = data + (size_t)lst[local * nb + r] * BT_ROW;
            if (jit) {  // one uniform per row (sampling.py:168-170)
              const uint64_t w = derive5(TAG_DATA_WORKER, a.seed, (uint64_t)epoch, (uint64_t)local, (uint64_t)eg);
              ju = dmul(dsub(unit_float(draw_raw(w, (uint64_t)r)), 0.5), a.jitter);
            }
          }
#pragma unroll
          for (int i = 0; i < BT_ROW; ++i) x[i] = src[i];
        }
        const long long tb0 = L.timing ? clock64() : 0;
#pragma unroll
        for (int i = 0; i < BT_INPUT_DIM; ++i) x[i] = jit ? dadd(x[i], ju) : x[i];
        {  // lane j < 8 keeps input j, lane 8 keeps y: a select chain, no divergent stores
          double keepv = x[0];
#pragma unroll
          for (int i = 1; i < BT_ROW; ++i) keepv = j == i ? x[i] : keepv;
          if (valid && j < BT_INPUT_DIM) s_x[row * BT_INPUT_DIM + j] = keepv;
          else if (valid && j == BT_INPUT_DIM) s_y[row] = keepv;
        }
        double acc = dmul(s_par[BT_W1 + j], x[0]);
#pragma unroll
        for (int i = 1; i < BT_INPUT_DIM; ++i) acc = dadd(acc, dmul(s_par[BT_W1 + i * BT_HIDDEN + j], x[i]));
        const double pre = dadd(acc, s_par[BT_B1 + j]);
        long long tb1 = 0;
        if (L.timing && tid == 0) {  // profiling: keep `pre` live before the clock read
          asm volatile("" ::"d"(pre));
          tb1 = clock64();
        }
        const double act = glibc_tanh_simt(pre);
        if (L.timing && tid == 0) {
          asm volatile("" ::"d"(act));
          const long long tb2 = clock64();
          tacc[6] += (unsigned long long)(tb1 - tb0);
          tacc[7] += (unsigned long long)(tb2 - tb1);
          tacc[8] += (unsigned long long)(tb0 - tlast);
        }
        double m = 1.0;
        if (rate > 0.0) {  // draw n = r*16+j of this EST's stream (rows outer, units inner)
          const double ud = unit_float(draw_raw(s_rng[el], (uint64_t)(r * BT_HIDDEN + j)));
          m = ud < rate ? 0.0 : keep;
        }
        const double hj = dmul(act, m);
        if (valid) {
          s_act[it] = act;
          s_hid[it] = hj;
        }
        __syncwarp();
        // C (lanes of invalid rows recompute row 0 and store nothing)
        const double* h = s_hid + row * BT_HIDDEN;
        const double* ar = s_act + row * BT_HIDDEN;
        double acc2 = dmul(s_par[BT_W2], h[0]);
        double msum = ar[0];
#pragma unroll
        for (int q = 1; q < BT_HIDDEN; ++q) {
          acc2 = dadd(acc2, dmul(s_par[BT_W2 + q], h[q]));
          msum = dadd(msum, ar[q]);
        }
        if (valid) {
          const double err = dsub(dadd(acc2, s_par[BT_B2]), s_y[row]);
          const double gy = divB.apply(dmul(2.0, err));
          s_dz[it] = dmul(dmul(dmul(gy, s_par[BT_W2 + j]), m), dsub(1.0, dmul(act, act)));
          if (j == 0) {
            s_e2[row] = dmul(err, err);
            s_gy[row] = gy;
            s_rm[row] = divH.apply(msum);
          }
        }
      }
    }
    __syncthreads();
    BT_TICK(0)

    // ---- E: per-EST gradients -> EST slot; loss, TrackedStat, RNG ---------
    // One thread per (EST, parameter): a batch-dim reduce_sum in the EST's
    // executor variant over precomputed terms (model.py:183-192) -- short
    // independent chains, because with a few warps per SM the step is
    // latency-bound and per-thread instruction count is the cost.  One more
    // thread per EST folds the loss and updates TrackedStat and the RNG.
    double* gbuf = a.grads + (a.fuse_reduce ? (size_t)par * (size_t)a.E * BT_P : 0);
    const bool to_global = !a.fuse_reduce || G > 1;
    if (L.cluster && tid == 0) mbar_arrive_expect_tx(smem_u32(&s_mbar[par]), slot_bytes);
    constexpr int ITEMS = BT_P + 1;
#pragma unroll 1
    for (int it = tid; it < ne * ITEMS; it += T) {
      const int el = it / ITEMS, p = it - el * ITEMS;
      const int rb = el * nb;
      const int fan = FB >= 0 ? FB : s_fan[el];
      const double g = fold_rows<BT, FB>(nb, fan, [&](int r) {
        const int row = rb + r;
        if (p < BT_B1) return dmul(s_dz[row * BT_HIDDEN + (p & 15)], s_x[row * BT_INPUT_DIM + (p >> 4)]);  // w1
        if (p < BT_W2) return s_dz[row * BT_HIDDEN + (p - BT_B1)];                                         // b1
        if (p < BT_B2) return dmul(s_gy[row], s_hid[row * BT_HIDDEN + (p - BT_W2)]);                      // w2
        if (p == BT_B2) return s_gy[row];                                                                  // b2
        return s_e2[row];                                                                                  // loss
      });
      if (p < BT_P) {
        if (L.cluster) {  // push this EST's slot into every CTA's copy of the step-parity slot array
          const uint32_t off = (uint32_t)((((size_t)par * Et + e0 + el) * BT_P + p) * sizeof(double));
          for (int rk = 0; rk < G; ++rk) st_async_f64(s_peer[rk] + off, g, s_peerbar[rk] + par * 8);
        } else if (to_global) {
          gbuf[(size_t)(e0 + el) * BT_P + p] = g;
        } else if (L.grads_smem) {
          s_grad[(size_t)(e0 + el) * BT_P + p] = g;
        }
      } else {
        const int e = e0 + el;
        const double loss = divB.apply(g);
        a.losses[(size_t)s * a.E + e] = loss;
        double bm = s_rm[rb];
        for (int r = 1; r < nb; ++r) bm = dadd(bm, s_rm[rb + r]);
        bm = divB.apply(bm);
        const int64_t rank = a.rank_override >= 0 ? a.rank_override : (int64_t)(a.est_base + e);
        const double mixed = dadd(bm, dmul((double)rank, 0x1p-40));  // model.py:99-104
        s_mean[el] = dadd(dmul(s_mean[el], 0.9), dmul(0.1, mixed));
        s_cnt[el] += 1;
        if (rate > 0.0) s_rng[el] = advance(s_rng[el], (uint64_t)nb * BT_HIDDEN);
      }
    }
    if (!a.fuse_reduce) {  // grads-only mode (K == 1): the host reduces
      ++s;
      break;
    }
    BT_TICK(1)

    // ---- exchange: every EST slot of this step in local shared memory -----
    if (L.cluster) {
      // Wait for all E_total*P*8 bytes of step parity `par` (peers' st.async
      // complete_tx; acquire).  A CTA is at most one step ahead of any peer:
      // its step s+1 pushes need every peer's step s+1 slots, which each
      // peer only pushes after finishing its step-s fold -- so the parity
      // double buffer is never overwritten while being read.
      const uint32_t bar = smem_u32(&s_mbar[par]);
      const uint32_t want = (phases >> par) & 1u;
      if (!mbar_try_wait(bar, want)) {
        const long long t0 = clock64();
        while (!mbar_try_wait(bar, want)) {
          if (clock64() - t0 > (1ll << 34)) {  // ~9 s: a lost arrival is a bug; fail instead of hanging
            atomicCAS(a.flags + FLAG_STATUS, 0, (int)ERR_CUDA);
            __trap();
          }
        }
      }
      phases ^= 1u << par;
    } else {
      if (G > 1) {
        if (!grid_sync(a.bar, (uint32_t)(s + 1) * (uint32_t)G, a.flags)) break;
        for (int i = tid; i < Et * BT_P; i += T) s_grad[i] = __ldcg(gbuf + i);  // L2: other CTAs' slots
      }
      __syncthreads();
    }
    BT_TICK(2)

    // ---- F: fixed-order allreduce + /E + momentum SGD into the next buffers
    // Leaf k of parameter p is EST slot (rot[p] + k) mod E: ascending virtual
    // rank, rotated by the parameter's ring chunk under Tree (buckets.py:115-123).
    int ok = 1;
    double np = 0.0;
    const int p = tid;
    if (p < BT_P) {
      const double* col = s_grad + (L.cluster ? (size_t)par * Et * BT_P : 0) + p;
      auto ld = [&](int q) { return col[(size_t)q * BT_P]; };
      double sum;
      if constexpr (SPEC) sum = fold_ranks_t<ET, FC>(s_rot[p], ld);
      else sum = fold_ranks_any(Et, a.comm_fanin, s_rot[p], ld);
      const double g = divE.apply(sum);
      ok = finite_d(g) ? 1 : 0;
      const double v = dadd(dmul(a.mu, s_vel[p]), g);
      np = dsub(s_par[p], dmul(a.lr, v));
      s_vel_n[p] = v;
      s_par_n[p] = np;
    }
    BT_TICK(3)
    if (!__syncthreads_and(ok)) {  // sgd_step raises before mutating (model.py:207-209)
      if (cta == 0 && tid == 0) {
        a.flags[FLAG_STATUS] = ERR_NUMERIC;
        a.flags[FLAG_STEP] = s;
      }
      break;  // this mini-batch's EST contexts already advanced (engine.py:301-302)
    }
    {  // commit: the next buffers become current
      double* t = s_par;
      s_par = s_par_n;
      s_par_n = t;
      t = s_vel;
      s_vel = s_vel_n;
      s_vel_n = t;
    }
    if (a.param_trace && cta == 0 && p < BT_P) a.param_trace[(size_t)s * BT_P + p] = np;
    BT_TICK(4)
  }
  if (L.timing && tid == 0 && cta == 0) {
    for (int k = 0; k < 5; ++k) L.timing[k] += tacc[k];
    for (int k = 6; k < 9; ++k) L.timing[k] += tacc[k];
    L.timing[5] += (unsigned long long)s;
  }

  // ---- epilogue: EST slots back to HBM; mirror the update to every replica
  if (L.cluster) cluster_barrier();  // no CTA leaves while a peer may still address it
  else __syncthreads();
  for (int el = tid; el < ne; el += T) {
    a.rng[e0 + el] = s_rng[el];
    a.stat_mean[e0 + el] = s_mean[el];
    a.stat_count[e0 + el] = s_cnt[el];
  }
  // (after a NumericError s_par holds the last successfully updated parameters)
  if (a.fuse_reduce && cta == 0) {  // engine.py:313-315
    for (int x = 0; x < a.X; ++x) {
      double* rx = a.replicas + (size_t)x * 2 * BT_P;
      for (int i = tid; i < BT_P; i += T) {
        rx[i] = s_par[i];
        rx[BT_P + i] = s_vel[i];
      }
    }
  }
}

// ---------------------------------------------------------------------------
// Compact build for the common shapes: B = 4 rows per EST, E_total = ET in
// {4, 8, 16} ESTs on one thread-block cluster of G CTAs (default min(ET, 8); EPC =
// ET / G ESTs each), one reduction variant F (0 = Sequential, 2 = Tree(2))
// for every EST's batch reductions and for the allreduce, dataset and index
// lists (or, for an explicit global batch, this CTA's rows) staged in shared memory.  Same arithmetic, same order as the generic
// build; what changes is the bookkeeping: the shared-memory layout and every
// thread's role are compile-time, each thread's addresses (rows, gradient
// operands, DSMEM push targets, allreduce leaves) are computed once per
// launch, and the next mini-batch's row gather, jitter and dropout mask are
// prefetched while the slot exchange is in flight.
// Exchange: all-to-all of the EST gradient slots (own slot by local store,
// peers' by st.async counted on the receiver's mbarrier) and a redundant,
// bit-identical stage F in every CTA.  An owner-computes reduce-scatter +
// all-gather moves 4x fewer DSMEM bytes but needs a second exchange per step;
// measured on B200 it is ~10% slower (the exchange is latency-bound, ~500
// cycles per hop), so one hop wins.
template <int ET, int GG, int ND = 1>
struct SpecShape {
  static constexpr int G = GG;                                           // CTAs = cluster size
  static constexpr int EL = ET / ND;                                     // ESTs on this device
  static constexpr int EPC = EL / G;                                     // ESTs per CTA
  static constexpr int SP = ND > 1 ? BT_XSP : BT_P;                      // slot stride (16-byte rows)
  static constexpr int GM1 = G > 1 ? G - 1 : 1;                          // (array extents)
  static constexpr int NB = 4;                                           // rows per EST
  static constexpr int R = NB * EPC;                                     // rows per CTA
  static constexpr int LANES = R * BT_HIDDEN;                            // stage B+C lanes
  static constexpr int T = LANES > 192 ? LANES : 192;                    // >= BT_P + 1
  static constexpr int ITEMS = EPC * (BT_P + 1);                         // stage E items
  static constexpr int NIT = (ITEMS + T - 1) / T;
  // shared-memory layout, in doubles
  static constexpr int PAR = 0;                    // [2][PAD_P] parameters (step-parity buffers)
  static constexpr int VEL = PAR + 2 * PAD_P;      // [2][PAD_P] velocity
  static constexpr int X = VEL + 2 * PAD_P;        // [R][8] jittered inputs
  static constexpr int Y = X + R * BT_INPUT_DIM;   // [R]
  static constexpr int ACT = Y + R;                // [R][16]
  static constexpr int HID = ACT + R * BT_HIDDEN;  // [R][16]
  static constexpr int DZ = HID + R * BT_HIDDEN;   // [R][16]
  static constexpr int GY = DZ + R * BT_HIDDEN;    // [R]
  static constexpr int E2 = GY + R;                // [R]
  static constexpr int RM = E2 + R;                // [R]
  static constexpr int MEAN = RM + R;              // [EPC]
  static constexpr int RNG = MEAN + EPC;           // [EPC] u64
  static constexpr int CNT = RNG + EPC;            // [EPC] u64
  static constexpr int GRAD = (CNT + EPC + 1) & ~1;  // [2][ET][SP] slot arrays (16-byte aligned)
  static constexpr int ROT = GRAD + 2 * ET * SP;     // int32 [PAD_P]
  static constexpr int DATA = ROT + PAD_P / 2;       // [dataset_rows][9], then jit [K][R], idx int32 [K][R]
  static constexpr size_t fixed_bytes() { return sizeof(double) * DATA; }
};

__device__ __forceinline__ void mbar_wait(uint32_t bar, uint32_t parity, int32_t* flags) {
  if (mbar_try_wait(bar, parity)) return;
  const long long t0 = clock64();
  while (!mbar_try_wait(bar, parity)) {
    if (clock64() - t0 > (1ll << 34)) {  // a lost arrival is a bug: fail instead of hanging
      atomicCAS(flags + FLAG_STATUS, 0, (int)ERR_CUDA);
      __trap();
    }
  }
}

__device__ __forceinline__ uint32_t ld_acquire_sys_u32(const uint32_t* p) {
  uint32_t v;
  asm volatile("ld.acquire.sys.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void red_release_sys_add(uint32_t* p, uint32_t v) {
  asm volatile("red.release.sys.global.add.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
__device__ __forceinline__ void fence_acq_rel_sys() { asm volatile("fence.acq_rel.sys;" ::: "memory"); }
// Flag-in-word ("LL") transfer of one binary64 across GPUs: two 8-byte words {32 data bits, 32-bit
// tag}, each written and read with single-copy-atomic 8-byte accesses, so a reader that sees the
// expected tag in both words holds the value -- no fence, no counter, no extra barrier.
__device__ __forceinline__ void ll_store(uint64_t* p, double v, uint32_t tag) {
  const uint64_t u = d2u(v), t = (uint64_t)tag << 32;
  asm volatile("st.volatile.global.v2.u64 [%0], {%1, %2};" ::"l"(p), "l"((u & 0xffffffffull) | t), "l"((u >> 32) | t)
               : "memory");
}
__device__ __forceinline__ void ll_load_raw(const uint64_t* p, uint64_t* w0, uint64_t* w1) {
  asm volatile("ld.volatile.global.v2.u64 {%0, %1}, [%2];" : "=l"(*w0), "=l"(*w1) : "l"(p) : "memory");
}
__device__ __forceinline__ bool ll_ready(uint64_t w0, uint64_t w1, uint32_t tag) {
  return (uint32_t)(w0 >> 32) == tag && (uint32_t)(w1 >> 32) == tag;
}
__device__ __forceinline__ double ll_value(uint64_t w0, uint64_t w1) {
  return __longlong_as_double((long long)((w0 & 0xffffffffull) | (w1 << 32)));
}

// The launch's losses and the 4 status words (the one-copy layout) into mapped host memory, then the done
// word with a system-scope release (all threads of one CTA; bt_mlp_run spins on the word).
__device__ __forceinline__ void spec_signal_host(const bt_mlp_args& a, const MlpLaunch& L, int tid, int T) {
  const int nw = a.K * a.E_total + 2;
  const unsigned long long* src = (const unsigned long long*)a.losses;
  unsigned long long* dst = (unsigned long long*)L.host_out;
  for (int i = tid; i < nw; i += T) dst[i] = __ldcg(src + i);
  __threadfence_system();
  __syncthreads();
  if (tid == 0) asm volatile("st.release.sys.global.u32 [%0], %1;" ::"l"(L.host_done), "r"(L.done_seq) : "memory");
}

template <int ET, int G, int F, int ND = 1>
__global__ void __launch_bounds__(SpecShape<ET, G, ND>::T) mlp_step_spec_kernel(const __grid_constant__ bt_mlp_args a,
                                                                                 const MlpLaunch L) {
  using S = SpecShape<ET, G, ND>;
  static_assert((G > 1 || ND > 1) && ET % (G * ND) == 0, "compact build: a cluster of G CTAs per device");
  extern __shared__ __align__(16) double sm[];
  const int tid = threadIdx.x;
  const int cta = blockIdx.x;  // the grid is one cluster: blockIdx.x is the cluster rank
  const int e0 = cta * S::EPC;
  const int eb = ND > 1 ? a.est_base : 0;  // global rank of this device's first EST
  // sampler mode: the resident dataset + this launch's (index, jitter) per row;
  // explicit-batch mode (split_by_rank rows, engine.py:261-268): this CTA's own
  // rows of every mini-batch, index = position, jitter = 0 (rows are final)
  const int64_t data_rows = a.rows ? (int64_t)a.K * S::R : a.dataset_rows;
  double* const s_data = sm + S::DATA;
  double* const s_jit = s_data + (size_t)data_rows * BT_ROW;
  int32_t* const s_idx = (int32_t*)(s_jit + (size_t)a.K * S::R);
  int32_t* const s_rot = (int32_t*)(sm + S::ROT);
  uint64_t* const s_rng = (uint64_t*)(sm + S::RNG);
  uint64_t* const s_cnt = (uint64_t*)(sm + S::CNT);
  __shared__ __align__(8) uint64_t s_mbar[3];  // [0], [1]: slot exchange by step parity; [2]: dataset
  const long long t_entry = clock64();

  // ---- prologue: everything below is issued at once and overlaps ---------
  // Sampler mode: the resident dataset arrives in one bulk copy per CTA (the copy engine streams
  // it while the threads fetch the parameters, slots and index lists); the cluster barrier that
  // orders every CTA's mbarrier initialisation before the first DSMEM push is split around the
  // prologue (arrive now, wait before the loop), so it costs nothing on the critical path.
  const int64_t nd_bytes = a.rows ? 0 : a.dataset_rows * BT_ROW * (int64_t)sizeof(double);
  const bool bulk = nd_bytes > 0 && (nd_bytes & 15) == 0 && (((uintptr_t)a.dataset) & 15) == 0 &&
                    nd_bytes < (1 << 20);
  if (tid == 0) {  // a phase completes when every local thread arrived and every remote byte landed
    mbar_init(smem_u32(&s_mbar[0]), S::T);
    mbar_init(smem_u32(&s_mbar[1]), S::T);
    mbar_init(smem_u32(&s_mbar[2]), 1);
    mbar_init_fence();
    if (bulk) {
      const uint32_t bar = smem_u32(&s_mbar[2]);
      mbar_arrive_expect_tx(bar, (uint32_t)nd_bytes);
      bulk_g2s(smem_u32(s_data), a.dataset, (uint32_t)nd_bytes, bar);
    }
  }
  cluster_arrive();
  const long long t_p0 = clock64();
  // Every global load of the prologue is issued before any is consumed (one HBM round trip after the
  // L2 is cold, not three): the status word, this thread's parameters / velocity / rotation entries, its
  // EST-slot and variant-hint words and (sampler mode) its first IPT index-list entries.
  const int flag0 = a.flags[FLAG_STATUS];
  constexpr int PPT = (BT_P + S::T - 1) / S::T, IPT = 4;
  double pp[PPT], pv[PPT];
  int32_t pr[PPT];
#pragma unroll
  for (int k = 0; k < PPT; ++k) {
    const int i = tid + k * S::T;
    if (i < BT_P) {
      pp[k] = a.replicas[i];
      pv[k] = a.replicas[BT_P + i];
      pr[k] = a.rot ? a.rot[i] : 0;
    }
  }
  uint64_t l_rng = 0, l_cnt = 0;
  double l_mean = 0.0;
  if (tid < S::EPC) {
    l_rng = a.rng[e0 + tid];
    l_mean = a.stat_mean[e0 + tid];
    l_cnt = a.stat_count[e0 + tid];
  }
  const int l_fan = tid < S::EL ? a.est_fanin[tid] : F;
  const int64_t ep0 = a.spe > 0 ? a.step0 / a.spe : 0;
  const int spe = (int)a.spe, loc0 = (int)(a.step0 - ep0 * a.spe);
  auto list_entry = [&](int it) -> const int32_t* {  // (mini-batch s, row) -> its index-list entry
    const int s = it / S::R, rem = it - s * S::R;
    const int el = rem / S::NB, r = rem - el * S::NB;
    const int q = loc0 + s, de = q / spe, local = q - de * spe;
    return a.lists + ((size_t)(ep0 + de - a.epoch_base) * ET + (eb + e0 + el)) * (size_t)(spe * S::NB) +
           local * S::NB + r;
  };
  int32_t iv[IPT];
  if (!a.rows) {
#pragma unroll
    for (int k = 0; k < IPT; ++k) {
      const int it = tid + k * S::T;
      if (it < a.K * S::R) iv[k] = *list_entry(it);
    }
  }
  if (!a.rows) {  // the rows' jitter needs only counters: computed while the loads above are in flight
    for (int it = tid; it < a.K * S::EPC; it += S::T) {  // one worker stream per (mini-batch, EST)
      const int s = it / S::EPC, el = it - s * S::EPC;
      const int q = loc0 + s, de = q / spe, local = q - de * spe;
      double* jd = s_jit + (size_t)s * S::R + el * S::NB;
      if (a.jitter != 0.0) {  // one uniform per row of worker_rng(seed, epoch, local, est) (sampling.py:99-170)
        const uint64_t w = derive5(TAG_DATA_WORKER, a.seed, (uint64_t)(ep0 + de), (uint64_t)local, (uint64_t)(eb + e0 + el));
#pragma unroll
        for (int r = 0; r < S::NB; ++r) jd[r] = dmul(dsub(unit_float(draw_raw(w, (uint64_t)r)), 0.5), a.jitter);
      } else {
#pragma unroll
        for (int r = 0; r < S::NB; ++r) jd[r] = 0.0;
      }
    }
  }
  // ---- per-thread constants (pure arithmetic: computed while the prologue's loads are in flight) ----
  const double rate = a.rate, lr = a.lr, mu = a.mu;
  const double keep = rate >= 1.0 ? 0.0 : ddiv(1.0, dsub(1.0, rate));  // model.py:150
  const bool jit = !a.rows && a.jitter != 0.0;
  const IntDivisor divB = IntDivisor::of(S::NB), divH = IntDivisor::of(BT_HIDDEN), divE = IntDivisor::of(ET);
  // B+C lane: row = tid / 16 of this CTA, hidden unit j = tid % 16
  const bool lane = tid < S::LANES;
  const int row = lane ? tid >> 4 : 0, j = tid & 15;
  const int lel = row / S::NB, lr_ = row - lel * S::NB;
  // E items: (EST, parameter or loss) pairs.  Term r of item (el, p) is
  // A[r] * B[r] (w1: dz*x, w2: gy*h) or A[r] (b1: dz, b2: gy, loss: e^2);
  // the operand addresses are per-thread constants, so the step's gradient
  // code is loads, multiplies, a select and the fold -- no branches.
  uint32_t opa[S::NIT][S::NB], opb[S::NIT][S::NB], own_dst[S::NIT], rdst[S::NIT][S::GM1];
  bool has_b[S::NIT], is_loss[S::NIT], valid[S::NIT];
  uint32_t rbar[S::GM1];
  const uint32_t sm0 = smem_u32(sm);
#pragma unroll
  for (int i = 0; i < G - 1; ++i) {  // the other CTAs, in rotated order (no rank test per push)
    int rk = cta + 1 + i;
    rk -= rk >= G ? G : 0;
    rbar[i] = cluster_map32(smem_u32(&s_mbar[0]), rk);
  }
#pragma unroll
  for (int k = 0; k < S::NIT; ++k) {
    const int it = tid + k * S::T;
    valid[k] = it < S::ITEMS;
    const int el = valid[k] ? it / (BT_P + 1) : 0, p = valid[k] ? it - el * (BT_P + 1) : 0;
    const int rb = el * S::NB;
    int a0, as, b0, bs;  // first operand index and row stride, in doubles
    if (p < BT_B1) { a0 = S::DZ + rb * BT_HIDDEN + (p & 15); as = BT_HIDDEN; b0 = S::X + rb * BT_INPUT_DIM + (p >> 4); bs = BT_INPUT_DIM; }
    else if (p < BT_W2) { a0 = S::DZ + rb * BT_HIDDEN + (p - BT_B1); as = BT_HIDDEN; b0 = a0; bs = as; }
    else if (p < BT_B2) { a0 = S::GY + rb; as = 1; b0 = S::HID + rb * BT_HIDDEN + (p - BT_W2); bs = BT_HIDDEN; }
    else if (p == BT_B2) { a0 = S::GY + rb; as = 1; b0 = a0; bs = as; }
    else { a0 = S::E2 + rb; as = 1; b0 = a0; bs = as; }
    has_b[k] = p < BT_W2 ? p < BT_B1 : p < BT_B2;
    is_loss[k] = p == BT_P;
#pragma unroll
    for (int r = 0; r < S::NB; ++r) {
      opa[k][r] = sm0 + (uint32_t)((a0 + r * as) * sizeof(double));
      opb[k][r] = sm0 + (uint32_t)((b0 + r * bs) * sizeof(double));
    }
    const uint32_t off = (uint32_t)((S::GRAD + (eb + e0 + el) * S::SP + p) * sizeof(double));  // parity-0 slot entry
    own_dst[k] = sm0 + off;
#pragma unroll
    for (int i = 0; i < G - 1; ++i) {
      int rk = cta + 1 + i;
      rk -= rk >= G ? G : 0;
      rdst[k][i] = cluster_map32(sm0, rk) + off;
    }
  }
  int bad = flag0 != 0 ? 4 : 0;  // a sticky earlier failure: do nothing
#pragma unroll
  for (int k = 0; k < PPT; ++k) {
    const int i = tid + k * S::T;
    if (i < BT_P) {
      sm[S::PAR + i] = pp[k];
      sm[S::VEL + i] = pv[k];
      s_rot[i] = pr[k];
      for (int x = 1; x < a.X; ++x) {  // replica agreement, bytewise (engine.py:246-258)
        const double* rx = a.replicas + (size_t)x * 2 * BT_P;
        bad |= (d2u(rx[i]) != d2u(pp[k])) | (d2u(rx[BT_P + i]) != d2u(pv[k]));
      }
    }
  }
  if constexpr (ND > 1) {  // every device's first replica against ours: all devices see the same verdict
    for (int i = tid; i < 2 * BT_P; i += S::T) {
      const uint64_t mine = d2u(a.replicas[i]);
#pragma unroll
      for (int q = 0; q < ND; ++q)
        if (a.xrep[q]) bad |= d2u(__ldcg(a.xrep[q] + i)) != mine;
    }
  }
  if (tid < S::EPC) {
    s_rng[tid] = l_rng;
    sm[S::MEAN + tid] = l_mean;
    s_cnt[tid] = l_cnt;
  }
  // the launcher's variant hint must hold -- checked for every EST in every CTA, so the whole
  // cluster takes the same exit
  bad |= (l_fan != F) << 1;
  const long long t_p1 = clock64();
  long long t_p2 = t_p1;
  if (a.rows) {
    for (int it = tid; it < a.K * S::R; it += S::T) {
      const int s = it / S::R, rem = it - s * S::R;
      const int el = rem / S::NB, r = rem - el * S::NB;
      const double* src = a.rows + ((size_t)s * S::NB * ET + (size_t)r * ET + (eb + e0 + el)) * BT_ROW;
#pragma unroll
      for (int i = 0; i < BT_ROW; ++i) s_data[(size_t)it * BT_ROW + i] = src[i];
      s_idx[it] = it;
      s_jit[it] = 0.0;
    }
  } else {
    if (!bulk) {
      const int64_t nd = a.dataset_rows * BT_ROW;
      for (int64_t i = tid; i < nd; i += S::T) s_data[i] = a.dataset[i];
    }
#pragma unroll
    for (int k = 0; k < IPT; ++k) {
      const int it = tid + k * S::T;
      if (it < a.K * S::R) s_idx[it] = iv[k];
    }
#pragma unroll 4
    for (int it = tid + IPT * S::T; it < a.K * S::R; it += S::T) s_idx[it] = *list_entry(it);  // long launches
    t_p2 = clock64();
  }
  const long long t_p3 = clock64();
  if (bulk) mbar_wait(smem_u32(&s_mbar[2]), 0, a.flags);  // the dataset has landed (also before any exit)
  const long long t_p4 = clock64();
  const int prologue = __syncthreads_or(bad);
  const long long t_p5 = clock64();
  cluster_wait();  // every CTA's mbarriers are initialised (and every CTA took the same branch below)
  if (prologue) {  // identical in every CTA of the cluster
    if (cta == 0 && tid == 0 && !(prologue & 4)) {
      a.flags[FLAG_STATUS] = (prologue & 1) ? ERR_CORRUPTION : ERR_INPUT;
      a.flags[FLAG_STEP] = 0;
    }
    if constexpr (ND == 1) {
      if (L.host_out && cta == 0) {  // the host waits on the signal: publish the status words
        __threadfence();
        __syncthreads();
        spec_signal_host(a, L, tid, S::T);
      }
    }
    return;
  }

  uint64_t lrng = s_rng[lel];  // this row's EST dropout stream, advanced in registers
  const int rot_p = tid < BT_P ? s_rot[tid] : 0;
  uint32_t phases = 0;

  // prefetched inputs of the next mini-batch (lane threads)
  double x[BT_ROW], msk = 1.0;
  auto prefetch = [&](int s) {
    const int q = s * S::R + row;
    const double* src = s_data + (size_t)s_idx[q] * BT_ROW;
    const double ju = s_jit[q];
#pragma unroll
    for (int i = 0; i < BT_INPUT_DIM; ++i) x[i] = jit ? dadd(src[i], ju) : src[i];
    x[BT_INPUT_DIM] = src[BT_INPUT_DIM];
    msk = 1.0;
    if (rate > 0.0) {  // draw n = r*16+j of this EST's stream (rows outer, units inner)
      const double ud = unit_float(draw_raw(lrng, (uint64_t)(lr_ * BT_HIDDEN + j)));
      msk = ud < rate ? 0.0 : keep;
    }
  };
  if (lane) prefetch(0);

  unsigned long long tacc[9] = {0, 0, 0, 0, 0, 0, 0, 0, 0};
  long long tlast = clock64();
  const long long t_loop = tlast;
  int cur = 0, s = 0;
  for (; s < a.K; ++s) {
    const int par = (int)((a.step0 + s) & 1);
    const uint32_t xtag = (uint32_t)(a.step0 + s + 1);  // (multi-device) tag of this mini-batch's slots
    const double* P = sm + S::PAR + cur * PAD_P;

    // ---- B+C (model.py:141-179, 194) --------------------------------------
    if (lane) {
      {  // lane j < 8 keeps input j, lane 8 keeps y
        double keepv = x[0];
#pragma unroll
        for (int i = 1; i < BT_ROW; ++i) keepv = j == i ? x[i] : keepv;
        if (j < BT_INPUT_DIM) sm[S::X + row * BT_INPUT_DIM + j] = keepv;
        else if (j == BT_INPUT_DIM) sm[S::Y + row] = keepv;
      }
      double acc = dmul(P[BT_W1 + j], x[0]);
#pragma unroll
      for (int i = 1; i < BT_INPUT_DIM; ++i) acc = dadd(acc, dmul(P[BT_W1 + i * BT_HIDDEN + j], x[i]));
#if defined(BT_ABL) && (BT_ABL & 1)  // timing ablation builds only (tools/ablate.sh)
      const double act = dadd(acc, P[BT_B1 + j]);
#else
      const double act = glibc_tanh_simt(dadd(acc, P[BT_B1 + j]));
#endif
      const double hj = dmul(act, msk);
      sm[S::ACT + tid] = act;
      sm[S::HID + tid] = hj;
      __syncwarp();
      const double* h = sm + S::HID + row * BT_HIDDEN;
      const double* ar = sm + S::ACT + row * BT_HIDDEN;
      double o = dmul(P[BT_W2], h[0]);
      double msum = ar[0];
#pragma unroll
      for (int q = 1; q < BT_HIDDEN; ++q) {
        o = dadd(o, dmul(P[BT_W2 + q], h[q]));
        msum = dadd(msum, ar[q]);
      }
      const double err = dsub(dadd(o, P[BT_B2]), x[BT_INPUT_DIM]);
      const double gy = divB.apply(dmul(2.0, err));
      sm[S::DZ + tid] = dmul(dmul(dmul(gy, P[BT_W2 + j]), msk), dsub(1.0, dmul(act, act)));
      if (j == 0) {
        sm[S::E2 + row] = dmul(err, err);
        sm[S::GY + row] = gy;
        sm[S::RM + row] = divH.apply(msum);
      }
    }
    __syncthreads();
    BT_TICK(0)

    // ---- E: gradients -> every CTA's slot array (model.py:183-192) --------
    const uint32_t pb = (uint32_t)(par * ET * S::SP * sizeof(double));  // step-parity slot array
#pragma unroll
    for (int k = 0; k < S::NIT; ++k) {
      if (valid[k]) {
        double v[S::NB];
#pragma unroll
        for (int r = 0; r < S::NB; ++r) {
          const double av = ld_shared_f64(opa[k][r]), bv = ld_shared_f64(opb[k][r]);
          v[r] = has_b[k] ? dmul(av, bv) : av;
        }
        const double g = TreeLevel<S::NB, F>::run(v);
        if (!is_loss[k]) {
          st_shared_f64(own_dst[k] + pb, g);  // own copy: a local store
#pragma unroll
          for (int i = 0; i < G - 1; ++i)
#if !(defined(BT_ABL) && (BT_ABL & 4))
            st_async_f64(rdst[k][i] + pb, g, rbar[i] + par * 8);
#else
            ;
#endif
          if constexpr (ND > 1) {  // the same value into every other device's inbox (NVLink stores)
            const int it = tid + k * S::T, el = it / (BT_P + 1), p = it - el * (BT_P + 1);
            const size_t off = ((size_t)(par * ET + eb + e0 + el) * S::SP + p) * 2;
#pragma unroll
            for (int r = 1; r < ND; ++r) {
              int d = a.dev_index + r;
              d -= d >= ND ? ND : 0;
              ll_store((uint64_t*)a.xin[d] + off, g, xtag);
            }
          }
        } else {  // loss, TrackedStat, dropout stream of EST e0+el (model.py:173, 99-104)
          const int el = (tid + k * S::T) / (BT_P + 1);
          const int e = eb + e0 + el, rb = el * S::NB;  // global rank
          a.losses[(size_t)s * ET + e] = divB.apply(g);
          double bm = sm[S::RM + rb];
#pragma unroll
          for (int r = 1; r < S::NB; ++r) bm = dadd(bm, sm[S::RM + rb + r]);
          bm = divB.apply(bm);
          const int64_t rank = a.rank_override >= 0 ? a.rank_override : (int64_t)e;
          const double mixed = dadd(bm, dmul((double)rank, 0x1p-40));
          sm[S::MEAN + el] = dadd(dmul(sm[S::MEAN + el], 0.9), dmul(0.1, mixed));
          s_cnt[el] += 1;
          if (rate > 0.0) s_rng[el] = advance(s_rng[el], (uint64_t)S::NB * BT_HIDDEN);
        }
      }
    }
    {  // local slot stores ordered before the arrival (release); thread 0 adds the remote bytes
      const uint32_t bar = smem_u32(&s_mbar[par]);
#if defined(BT_ABL) && (BT_ABL & 4)
      if (tid == 0) mbar_arrive_expect_tx(bar, 0);
#else
      if (tid == 0) mbar_arrive_expect_tx(bar, (uint32_t)((S::EL - S::EPC) * BT_P * sizeof(double)));
#endif
      else mbar_arrive(bar);
    }
    BT_TICK(1)
    // the next mini-batch's rows and masks while the exchange is in flight
    if (lane && s + 1 < a.K) {
      if (rate > 0.0) lrng = advance(lrng, (uint64_t)S::NB * BT_HIDDEN);
      prefetch(s + 1);
    }

    // ---- exchange: all ET*P*8 slot bytes of this step parity --------------
    mbar_wait(smem_u32(&s_mbar[par]), (phases >> par) & 1u, a.flags);
    phases ^= 1u << par;
    int xok = 1;
    BT_TICK(2)

    // ---- F: allreduce + /E + momentum SGD into the other buffer -----------
    int ok = 1;
    double np = 0.0;
    if (tid < BT_P) {
      const double* col = sm + S::GRAD + par * ET * S::SP + tid;
#if defined(BT_ABL) && (BT_ABL & 8)
      const double sum = col[0];
#else
      double sum;
      if constexpr (ND > 1) {  // the other devices' slots: poll each until its tag is this mini-batch's
        const uint64_t* inb = (const uint64_t*)a.xin[a.dev_index] + ((size_t)par * ET * S::SP + tid) * 2;
        double rv[ET];
        uint64_t w0[ET], w1[ET];
#pragma unroll
        for (int q = 0; q < ET; ++q)  // every remote value's first load in flight at once
          if ((unsigned)(q - eb) >= (unsigned)S::EL) ll_load_raw(inb + (size_t)q * S::SP * 2, &w0[q], &w1[q]);
#pragma unroll
        for (int q = 0; q < ET; ++q) {
          if ((unsigned)(q - eb) < (unsigned)S::EL) {
            rv[q] = col[q * S::SP];
            continue;
          }
          if (!ll_ready(w0[q], w1[q], xtag)) {  // not yet delivered: poll this one
            const long long tw = clock64();
            do {
              ll_load_raw(inb + (size_t)q * S::SP * 2, &w0[q], &w1[q]);
              if (clock64() - tw > (1ll << 32)) {  // a device that never delivers: fail, do not hang
                atomicCAS(a.flags + FLAG_STATUS, 0, (int)ERR_CUDA);
                xok = 0;
                break;
              }
            } while (!ll_ready(w0[q], w1[q], xtag));
          }
          rv[q] = ll_value(w0[q], w1[q]);
        }
        sum = fold_ranks_t<ET, F>(rot_p, [&](int q) { return rv[q]; });
      } else {
        sum = fold_ranks_t<ET, F>(rot_p, [&](int q) { return col[q * BT_P]; });
      }
#endif
      const double g = divE.apply(sum);
      ok = finite_d(g) ? 1 : 0;
      const double v = dadd(dmul(mu, sm[S::VEL + cur * PAD_P + tid]), g);
      np = dsub(P[tid], dmul(lr, v));
      sm[S::VEL + (cur ^ 1) * PAD_P + tid] = v;
      sm[S::PAR + (cur ^ 1) * PAD_P + tid] = np;
    }
    BT_TICK(3)
    if (!__syncthreads_and(ok && xok)) {  // sgd_step raises before mutating (model.py:207-209)
      if (cta == 0 && tid == 0 && a.flags[FLAG_STATUS] == 0) {
        a.flags[FLAG_STATUS] = ERR_NUMERIC;
        a.flags[FLAG_STEP] = s;
      }
      break;
    }
    cur ^= 1;
    if (a.param_trace && cta == 0 && tid < BT_P) a.param_trace[(size_t)s * BT_P + tid] = np;
    BT_TICK(4)
  }
  const long long t_loop_end = clock64();

  // ---- epilogue -----------------------------------------------------------
  // (every DSMEM push addressed to this CTA has landed -- its own mbarrier said so; the split
  // cluster barrier keeps each CTA resident until its peers are past their last push as well)
  cluster_arrive();
  for (int el = tid; el < S::EPC; el += S::T) {
    a.rng[e0 + el] = s_rng[el];
    a.stat_mean[e0 + el] = sm[S::MEAN + el];
    a.stat_count[e0 + el] = s_cnt[el];
  }
  if (cta == 0) {  // engine.py:313-315
    for (int x = 0; x < a.X; ++x) {
      double* rx = a.replicas + (size_t)x * 2 * BT_P;
      for (int i = tid; i < BT_P; i += S::T) {
        rx[i] = sm[S::PAR + cur * PAD_P + i];
        rx[BT_P + i] = sm[S::VEL + cur * PAD_P + i];
      }
    }
  }
  cluster_wait();
  if constexpr (ND == 1) {
    // every CTA's losses and status words are in global memory (cluster barrier)
    if (L.host_out && cta == 0) spec_signal_host(a, L, tid, S::T);
  }
  if (L.timing && tid == 0 && cta == 0) {  // [9] prologue, [10] epilogue, [11] whole CTA (cycles)
    for (int k = 0; k < 5; ++k) L.timing[k] += tacc[k];
    L.timing[5] += (unsigned long long)s;
    const long long t_exit = clock64();
    L.timing[9] += (unsigned long long)(t_loop - t_entry);
    L.timing[10] += (unsigned long long)(t_exit - t_loop_end);
    L.timing[11] += (unsigned long long)(t_exit - t_entry);
    // prologue detail: [6] init+issue, [7] params/slots loads, [8] index loads, [12] jitter,
    // [13] dataset wait, [14] CTA barrier, [15] cluster wait
    L.timing[6] += (unsigned long long)(t_p0 - t_entry);
    L.timing[7] += (unsigned long long)(t_p1 - t_p0);
    L.timing[8] += (unsigned long long)(t_p2 - t_p1);
    L.timing[12] += (unsigned long long)(t_p3 - t_p2);
    L.timing[13] += (unsigned long long)(t_p4 - t_p3);
    L.timing[14] += (unsigned long long)(t_p5 - t_p4);
    L.timing[15] += (unsigned long long)(t_loop - t_p5);
  }
}

static constexpr size_t SMEM_LIMIT = 220 * 1024;
static constexpr int SPEC_KCAP = 128;

static size_t base_smem_bytes(const bt_mlp_args& a) {
  const size_t rows = (size_t)a.est_per_cta * a.B;
  return sizeof(double) * (4 * PAD_P + rows * (BT_INPUT_DIM + 1 + 4 * BT_HIDDEN + 3) + 3 * (size_t)a.est_per_cta) +
         sizeof(int32_t) * (PAD_P + (((size_t)a.est_per_cta + 1) & ~(size_t)1));
}

static constexpr int MAX_CLUSTER = 8;  // portable cluster size

static int grid_of(const bt_mlp_args& a) { return (a.E + a.est_per_cta - 1) / a.est_per_cta; }

static bool use_cluster(const bt_mlp_args& a) {
  const int g = grid_of(a);
  return a.fuse_reduce && g > 1 && g <= MAX_CLUSTER &&
         base_smem_bytes(a) + sizeof(double) * 2 * (size_t)a.E_total * BT_P <= SMEM_LIMIT;
}

static MlpLaunch plan(const bt_mlp_args& a, size_t* smem) {
  MlpLaunch L{0, 0, 0, 0, nullptr};
  size_t bytes = base_smem_bytes(a);
  if (use_cluster(a)) {  // every CTA holds all [2][E][P] step-parity slots; peers push theirs via DSMEM
    L.cluster = 1;
    bytes += sizeof(double) * 2 * (size_t)a.E_total * BT_P;
  } else if (a.fuse_reduce) {
    const size_t g = sizeof(double) * (size_t)a.E_total * BT_P;
    if (bytes + g <= SMEM_LIMIT) {
      L.grads_smem = 1;
      bytes += g;
    }
  }
  if (!a.rows && a.dataset_rows > 0) {
    const size_t d = sizeof(double) * (size_t)a.dataset_rows * BT_ROW;
    if (bytes + d <= SMEM_LIMIT) {
      L.stage_data = 1;
      bytes += d;
    }
    const size_t ix = (sizeof(int32_t) + sizeof(double)) * (size_t)a.K * a.est_per_cta * a.B;  // idx + jitter
    if (bytes + ix <= SMEM_LIMIT) {
      L.stage_idx = 1;
      bytes += ix;
    }
  }
  *smem = bytes;
  return L;
}

size_t mlp_smem_bytes(int nrows) { return sizeof(double) * (4 * PAD_P + (size_t)nrows * 76); }

bool mlp_fused_fits(const bt_mlp_args& a) {
  if (a.E_total > BT_MAX_FUSED_E) return false;
  const size_t slots = use_cluster(a) ? 2 * (size_t)a.E_total : (size_t)a.E_total;
  return base_smem_bytes(a) + sizeof(double) * slots * BT_P <= SMEM_LIMIT;
}

template <class Kern>
static cudaError_t launch_cluster(Kern kern, const bt_mlp_args& a, size_t smem, int grid, int threads,
                                  cudaStream_t stream, const MlpLaunch& L) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(grid);
  cfg.blockDim = dim3(threads);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = stream;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = grid;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  return cudaLaunchKernelEx(&cfg, kern, a, L);
}

template <int BT>
static cudaError_t launch_k(const bt_mlp_args& a, const MlpLaunch& L, size_t smem, int grid, cudaStream_t stream) {
  static bool attr_set = false;  // one per instantiation
  if (!attr_set) {
    cudaError_t e =
        cudaFuncSetAttribute(mlp_step_kernel<BT>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)SMEM_LIMIT);
    if (e != cudaSuccess) return e;
    attr_set = true;
  }
  if (L.cluster) {
    // One cluster of `grid` CTAs on `grid` SMs; threads sized to the CTA's rows
    // (stage B: one thread per (row, unit)), at least one per parameter.
    int threads = ((a.est_per_cta * a.B * BT_HIDDEN + 31) / 32) * 32;
    threads = threads < 192 ? 192 : (threads > MLP_THREADS ? MLP_THREADS : threads);
    return launch_cluster(mlp_step_kernel<BT>, a, smem, grid, threads, stream, L);
  }
  if (grid > 1 && a.fuse_reduce) {
    if (cudaMemsetAsync(a.bar, 0, sizeof(uint32_t), stream) != cudaSuccess) return cudaGetLastError();
    void* params[] = {(void*)&a, (void*)&L};
    return cudaLaunchCooperativeKernel((const void*)mlp_step_kernel<BT>, dim3(grid), dim3(MLP_THREADS), params,
                                       smem, stream);
  }
  mlp_step_kernel<BT><<<grid, MLP_THREADS, smem, stream>>>(a, L);
  return cudaGetLastError();
}

template <int ET, int G, int F, int ND = 1>
static cudaError_t launch_spec(const bt_mlp_args& a, size_t smem, cudaStream_t stream, const MlpLaunch& L) {
  using S = SpecShape<ET, G, ND>;
  auto kern = mlp_step_spec_kernel<ET, G, F, ND>;
  static bool attr_set = false;
  if (!attr_set) {
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)SMEM_LIMIT);
    if (e != cudaSuccess) return e;
    attr_set = true;
  }
  return launch_cluster(kern, a, smem, G, S::T, stream, L);
}

// Shared memory of the compact build, or 0 when it does not fit.
template <int ET, int G, int ND = 1>
static size_t spec_smem(const bt_mlp_args& a) {
  using S = SpecShape<ET, G, ND>;
  const size_t data_rows = a.rows ? (size_t)a.K * S::R : (size_t)a.dataset_rows;
  // sampler mode: the per-launch (index, jitter) staging is sized for at least SPEC_KCAP
  // mini-batches, so launches of different lengths share one shared-memory configuration
  const size_t kst = a.rows ? (size_t)a.K : (size_t)(a.K > SPEC_KCAP ? a.K : SPEC_KCAP);
  const size_t bytes = S::fixed_bytes() + sizeof(double) * data_rows * BT_ROW +
                       (sizeof(double) + sizeof(int32_t)) * kst * S::R;
  if (bytes <= SMEM_LIMIT) return bytes;
  const size_t exact = S::fixed_bytes() + sizeof(double) * data_rows * BT_ROW +
                       (sizeof(double) + sizeof(int32_t)) * (size_t)a.K * S::R;
  return exact <= SMEM_LIMIT ? exact : 0;
}

template <int ET, int G, int ND = 1>
static bool try_spec(const bt_mlp_args& a, int fan, cudaStream_t stream, const MlpLaunch& L, cudaError_t* err) {
  const size_t ss = spec_smem<ET, G, ND>(a);
  if (!ss) return false;
  *err = fan ? launch_spec<ET, G, 2, ND>(a, ss, stream, L) : launch_spec<ET, G, 0, ND>(a, ss, stream, L);
  return true;
}

// Multi-device exchange group: E_total in {4, 8, 16} over n_dev in {2, 4, 8} devices, equal EST
// blocks, one cluster of min(E, 8) CTAs per device.
static bool try_spec_xdev(const bt_mlp_args& a, int fan, cudaStream_t stream, const MlpLaunch& L, cudaError_t* err) {
  switch (a.E_total * 16 + a.n_dev) {
    case 4 * 16 + 2: return try_spec<4, 2, 2>(a, fan, stream, L, err);
    case 4 * 16 + 4: return try_spec<4, 1, 4>(a, fan, stream, L, err);
    case 8 * 16 + 2: return try_spec<8, 4, 2>(a, fan, stream, L, err);
    case 8 * 16 + 4: return try_spec<8, 2, 4>(a, fan, stream, L, err);
    case 8 * 16 + 8: return try_spec<8, 1, 8>(a, fan, stream, L, err);
    case 16 * 16 + 2: return try_spec<16, 8, 2>(a, fan, stream, L, err);
    case 16 * 16 + 4: return try_spec<16, 4, 4>(a, fan, stream, L, err);
    case 16 * 16 + 8: return try_spec<16, 2, 8>(a, fan, stream, L, err);
    default: return false;
  }
}

bool mlp_xdev_supported(const bt_mlp_args& a) {
  const int fan = a.est_fanin_uniform - 1;
  const int ed = a.E_total * 16 + a.n_dev;
  const bool shape = ed == 4 * 16 + 2 || ed == 4 * 16 + 4 || ed == 8 * 16 + 2 || ed == 8 * 16 + 4 ||
                     ed == 8 * 16 + 8 || ed == 16 * 16 + 2 || ed == 16 * 16 + 4 || ed == 16 * 16 + 8;
  return shape && a.fuse_reduce && a.B == 4 && a.E * a.n_dev == a.E_total && a.est_base == a.dev_index * a.E &&
         (a.rows || a.dataset_rows > 0) && a.rank_override < 0 && (fan == 0 || fan == 2) && fan == a.comm_fanin;
}

// CTAs per cluster for the compact build (BT_SPEC_G overrides, for measurements).
static int spec_g(int et) {
  static int env = -1;
  if (env < 0) {
    const char* v = getenv("BT_SPEC_G");
    env = v ? atoi(v) : 0;
  }
  if (env > 0) return env;
  return et < 8 ? et : 8;
}

int mlp_launch(const bt_mlp_args& a, cudaStream_t stream, unsigned long long* timing, const MlpHostSignal* hs,
               bool* signaled) {
  if (signaled) *signaled = false;
  if (a.n_dev > 1) {  // one device of a lock-step exchange group: the compact build only
    if (!mlp_xdev_supported(a)) return ERR_INPUT;
    MlpLaunch L{0, 0, 0, 1, timing};
    cudaError_t err = cudaSuccess;
    if (!try_spec_xdev(a, a.est_fanin_uniform - 1, stream, L, &err)) return ERR_INPUT;
    return err == cudaSuccess ? OK : ERR_CUDA;
  }
  const int grid = grid_of(a);
  size_t smem = 0;
  MlpLaunch L = plan(a, &smem);
  L.timing = timing;
  const bool sig = hs && hs->out && hs->done && !timing;
  if (a.fuse_reduce && !L.grads_smem && !L.cluster) return ERR_INPUT;  // too many ESTs for the fused path
  if (smem > SMEM_LIMIT) return ERR_INPUT;
  const int fan = a.est_fanin_uniform - 1;  // every EST's batch variant, when the caller knows it
  if (a.fuse_reduce && a.B == 4 && a.E == a.E_total && (a.rows || a.dataset_rows > 0) && a.rank_override < 0 &&
      (fan == 0 || fan == 2) && fan == a.comm_fanin) {
    cudaError_t err = cudaSuccess;
    bool ran = false;
    const int g = spec_g(a.E_total);
    if (sig) {
      L.host_out = hs->out;
      L.host_done = hs->done;
      L.done_seq = hs->seq;
    }
    switch (a.E_total * 16 + g) {
      case 4 * 16 + 2: ran = try_spec<4, 2>(a, fan, stream, L, &err); break;
      case 4 * 16 + 4: ran = try_spec<4, 4>(a, fan, stream, L, &err); break;
      case 8 * 16 + 4: ran = try_spec<8, 4>(a, fan, stream, L, &err); break;
      case 8 * 16 + 8: ran = try_spec<8, 8>(a, fan, stream, L, &err); break;
      case 16 * 16 + 4: ran = try_spec<16, 4>(a, fan, stream, L, &err); break;
      case 16 * 16 + 8: ran = try_spec<16, 8>(a, fan, stream, L, &err); break;
      default: break;
    }
    if (ran) {
      if (signaled) *signaled = sig && err == cudaSuccess;
      return err == cudaSuccess ? OK : ERR_CUDA;
    }
    L.host_out = nullptr;  // (the generic build below does not signal)
    L.host_done = nullptr;
  }
  cudaError_t err;
  switch (a.B) {
    case 1: err = launch_k<1>(a, L, smem, grid, stream); break;
    case 2: err = launch_k<2>(a, L, smem, grid, stream); break;
    case 4: err = launch_k<4>(a, L, smem, grid, stream); break;
    case 8: err = launch_k<8>(a, L, smem, grid, stream); break;
    case 16: err = launch_k<16>(a, L, smem, grid, stream); break;
    case 32: err = launch_k<32>(a, L, smem, grid, stream); break;
    default: err = launch_k<0>(a, L, smem, grid, stream); break;
  }
  return err == cudaSuccess ? OK : ERR_CUDA;
}

}  // namespace bt
