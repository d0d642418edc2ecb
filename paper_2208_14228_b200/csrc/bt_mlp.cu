// bt_mlp.cu -- fused, persistent data-parallel step for the reference MLP.
//
// One launch runs K mini-batches of engine.run_minibatch (engine.py:271-329):
//   A  rows: device sampler (epoch lists + counter-form worker RNG jitter,
//      sampling.py:160-172) or an explicit global batch (split_by_rank,
//      engine.py:261-268);
//   B  hidden layer + tanh + dropout (model.py:141-163);
//   C  output error, loss terms, tracked-stat row means (model.py:165-176, 194);
//   D  dz, per-EST loss / TrackedStat / RNG advance (model.py:173-196, 99-104);
//   E  161 per-EST gradients, each a batch-dim reduce_sum in the EST's
//      executor variant (model.py:183-192) -> EST gradient slot;
//   F  the fixed-order allreduce in executor 0's variant (buckets.py:115-123,
//      rank order keyed by EST rank, never by GPU/CTA) fused with /E and the
//      momentum-SGD update (model.py:206-212).
// Layout: CTA c owns ESTs [c*epc, (c+1)*epc).  Stage F is computed by EVERY
// CTA redundantly (bit-identical: same inputs, same order), so a step needs a
// single grid barrier; gradient slots are double-buffered by step parity so a
// fast CTA's step s+1 writes never race a slow CTA's step s reads.
// Every binary64 op uses an explicit _rn intrinsic (no FMA contraction); tanh
// is glibc's (bt_libm.cuh), so results are bit-identical to the reference.
#include "bt_common.cuh"
#include "bt_libm.cuh"
#include "bt_mlp.cuh"

namespace bt {

constexpr int MLP_THREADS = 512;
constexpr int PAD_P = 168;  // 161 rounded up to a multiple of 8 doubles

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

__global__ void __launch_bounds__(MLP_THREADS) mlp_step_kernel(const __grid_constant__ bt_mlp_args a) {
  extern __shared__ __align__(16) double sm[];
  const int tid = threadIdx.x, T = blockDim.x;
  const int cta = blockIdx.x, G = gridDim.x;
  const int nb = a.B;
  const int e0 = cta * a.est_per_cta;
  const int ne = min(a.est_per_cta, a.E - e0);
  const int nrows = ne * nb;

  double* s_par = sm;
  double* s_vel = s_par + PAD_P;
  double* s_g = s_vel + PAD_P;
  double* s_x = s_g + PAD_P;                    // [nrows][8]
  double* s_y = s_x + nrows * BT_INPUT_DIM;     // [nrows]
  double* s_act = s_y + nrows;                  // [nrows][16] tanh outputs
  double* s_msk = s_act + nrows * BT_HIDDEN;    // [nrows][16] dropout masks
  double* s_hid = s_msk + nrows * BT_HIDDEN;    // [nrows][16] acts*mask
  double* s_dz = s_hid + nrows * BT_HIDDEN;     // [nrows][16]
  double* s_gy = s_dz + nrows * BT_HIDDEN;      // [nrows]
  double* s_e2 = s_gy + nrows;                  // [nrows]
  double* s_rm = s_e2 + nrows;                  // [nrows] row means of acts

  if (a.flags[FLAG_STATUS] != 0) return;  // sticky error from an earlier launch

  // Replica 0 into shared memory + replica agreement (engine.py:246-258: bytes).
  const double* rep0 = a.replicas;
  int bad = 0;
  // (grads-only mode needs no velocity: the seam passes a bare [161] params buffer)
  for (int i = tid; i < BT_P; i += T) {
    const double p0 = rep0[i];
    const double v0 = a.fuse_reduce ? rep0[BT_P + i] : 0.0;
    s_par[i] = p0;
    s_vel[i] = v0;
    for (int x = 1; x < a.X; ++x) {
      const double* rx = a.replicas + (size_t)x * 2 * BT_P;
      bad |= d2u(rx[i]) != d2u(p0);
      if (a.fuse_reduce) bad |= d2u(rx[BT_P + i]) != d2u(v0);
    }
  }
  if (__syncthreads_or(bad)) {
    if (cta == 0 && tid == 0) {
      a.flags[FLAG_STATUS] = ERR_CORRUPTION;
      a.flags[FLAG_STEP] = 0;
    }
    return;
  }

  const double rate = a.rate;
  const double keep = rate >= 1.0 ? 0.0 : ddiv(1.0, dsub(1.0, rate));  // model.py:150
  const double dB = (double)nb;

  for (int s = 0; s < a.K; ++s) {
    const int64_t gstep = a.step0 + s;
    const int64_t epoch = a.rows ? 0 : gstep / a.spe;
    const int64_t local = a.rows ? 0 : gstep % a.spe;

    // ---- A: micro-batch rows -------------------------------------------
    for (int it = tid; it < nrows; it += T) {
      const int el = it / nb, r = it - el * nb;
      const int eg = a.est_base + e0 + el;  // global virtual rank
      const double* src;
      double u = 0.0;
      bool jit = false;
      if (a.rows) {  // split_by_rank: row r of rank k is global row r*E+k
        src = a.rows + ((size_t)s * nb * a.E_total + (size_t)r * a.E_total + eg) * BT_ROW;
      } else {
        const int32_t* lst = a.lists + ((size_t)(epoch - a.epoch_base) * a.E_total + eg) * (size_t)(a.spe * nb);
        src = a.dataset + (size_t)lst[local * nb + r] * BT_ROW;
        if (a.jitter != 0.0) {  // one uniform per row (sampling.py:168-170)
          const uint64_t w = derive5(TAG_DATA_WORKER, a.seed, (uint64_t)epoch, (uint64_t)local, (uint64_t)eg);
          u = unit_float(draw_raw(w, (uint64_t)r));
          jit = true;
        }
      }
      const double ju = jit ? dmul(dsub(u, 0.5), a.jitter) : 0.0;
#pragma unroll
      for (int i = 0; i < BT_INPUT_DIM; ++i) {
        const double xv = src[i];
        s_x[it * BT_INPUT_DIM + i] = jit ? dadd(xv, ju) : xv;
      }
      s_y[it] = src[BT_INPUT_DIM];
    }
    __syncthreads();

    // ---- B: hidden pre-activation, tanh, dropout -------------------------
    for (int it = tid; it < nrows * BT_HIDDEN; it += T) {
      const int row = it >> 4, j = it & 15;
      const int el = row / nb, r = row - el * nb;
      const double* xr = s_x + row * BT_INPUT_DIM;
      double acc = dmul(s_par[BT_W1 + j], xr[0]);
#pragma unroll
      for (int i = 1; i < BT_INPUT_DIM; ++i) acc = dadd(acc, dmul(s_par[BT_W1 + i * BT_HIDDEN + j], xr[i]));
      const double act = glibc_tanh(dadd(acc, s_par[BT_B1 + j]));
      double m = 1.0;
      if (rate > 0.0) {  // draw n = r*16+j of this EST's stream (rows outer, units inner)
        const double ud = unit_float(draw_raw(a.rng[e0 + el], (uint64_t)(r * BT_HIDDEN + j)));
        m = ud < rate ? 0.0 : keep;
      }
      s_act[it] = act;
      s_msk[it] = m;
      s_hid[it] = dmul(act, m);
    }
    __syncthreads();

    // ---- C: output, error, upstream factor, row means --------------------
    for (int row = tid; row < nrows; row += T) {
      const double* h = s_hid + row * BT_HIDDEN;
      double acc = dmul(s_par[BT_W2], h[0]);
#pragma unroll
      for (int j = 1; j < BT_HIDDEN; ++j) acc = dadd(acc, dmul(s_par[BT_W2 + j], h[j]));
      const double err = dsub(dadd(acc, s_par[BT_B2]), s_y[row]);
      s_e2[row] = dmul(err, err);
      s_gy[row] = ddiv(dmul(2.0, err), dB);
      const double* ar = s_act + row * BT_HIDDEN;
      double m = ar[0];
#pragma unroll
      for (int j = 1; j < BT_HIDDEN; ++j) m = dadd(m, ar[j]);
      s_rm[row] = ddiv(m, (double)BT_HIDDEN);
    }
    __syncthreads();

    // ---- D: dz, loss, TrackedStat, RNG advance ---------------------------
    for (int it = tid; it < nrows * BT_HIDDEN; it += T) {
      const int row = it >> 4, j = it & 15;
      const double av = s_act[it];
      s_dz[it] = dmul(dmul(dmul(s_gy[row], s_par[BT_W2 + j]), s_msk[it]), dsub(1.0, dmul(av, av)));
    }
    for (int el = tid; el < ne; el += T) {
      const int e = e0 + el;
      StreamFold<double, 16> f;
      f.init(a.est_fanin[e]);
      for (int r = 0; r < nb; ++r) f.push(s_e2[el * nb + r]);
      a.losses[(size_t)s * a.E + e] = ddiv(f.finish(), dB);
      double bm = s_rm[el * nb];
      for (int r = 1; r < nb; ++r) bm = dadd(bm, s_rm[el * nb + r]);
      bm = ddiv(bm, dB);
      const int64_t rank = a.rank_override >= 0 ? a.rank_override : (int64_t)(a.est_base + e);
      const double mixed = dadd(bm, dmul((double)rank, 0x1p-40));  // model.py:99-104
      a.stat_mean[e] = dadd(dmul(a.stat_mean[e], 0.9), dmul(0.1, mixed));
      a.stat_count[e] += 1;
      if (rate > 0.0) a.rng[e] = advance(a.rng[e], (uint64_t)nb * BT_HIDDEN);
    }
    __syncthreads();

    // ---- E: per-EST gradients (batch-dim reduce_sum) -> EST slot ---------
    double* gbuf = a.grads + (a.fuse_reduce ? (size_t)(gstep & 1) * (size_t)a.E * BT_P : 0);
    for (int it = tid; it < ne * BT_P; it += T) {
      const int el = it / BT_P, p = it - el * BT_P;
      const int rb = el * nb;
      StreamFold<double, 16> f;
      f.init(a.est_fanin[e0 + el]);
      if (p < BT_B1) {
        const int i = p >> 4, j = p & 15;
        for (int r = 0; r < nb; ++r) f.push(dmul(s_dz[(rb + r) * BT_HIDDEN + j], s_x[(rb + r) * BT_INPUT_DIM + i]));
      } else if (p < BT_W2) {
        const int j = p - BT_B1;
        for (int r = 0; r < nb; ++r) f.push(s_dz[(rb + r) * BT_HIDDEN + j]);
      } else if (p < BT_B2) {
        const int j = p - BT_W2;
        for (int r = 0; r < nb; ++r) f.push(dmul(s_gy[rb + r], s_hid[(rb + r) * BT_HIDDEN + j]));
      } else {
        for (int r = 0; r < nb; ++r) f.push(s_gy[rb + r]);
      }
      gbuf[(size_t)(e0 + el) * BT_P + p] = f.finish();
    }
    if (!a.fuse_reduce) return;  // grads-only mode (K == 1): the host reduces

    // ---- F: fixed-order allreduce + /E + momentum SGD --------------------
    if (G > 1) {
      if (!grid_sync(a.bar, (uint32_t)(s + 1) * (uint32_t)G, a.flags)) return;
    } else {
      __syncthreads();
    }
    int ok = 1;
    const int Et = a.E_total;
    for (int p = tid; p < BT_P; p += T) {
      const int start = a.rot ? a.rot[p] : 0;
      StreamFold<double, 16> f;
      f.init(a.comm_fanin);
      for (int k = 0; k < Et; ++k) {
        int src = start + k;
        if (src >= Et) src -= Et;
        f.push(__ldcg(gbuf + (size_t)src * BT_P + p));  // L2: written by other CTAs this step
      }
      const double g = ddiv(f.finish(), (double)Et);
      s_g[p] = g;
      ok &= finite_d(g) ? 1 : 0;
    }
    if (!__syncthreads_and(ok)) {  // sgd_step raises before mutating (model.py:207-209)
      if (cta == 0 && tid == 0) {
        a.flags[FLAG_STATUS] = ERR_NUMERIC;
        a.flags[FLAG_STEP] = s;
      }
      return;
    }
    for (int p = tid; p < BT_P; p += T) {
      const double v = dadd(dmul(a.mu, s_vel[p]), s_g[p]);
      const double np = dsub(s_par[p], dmul(a.lr, v));
      s_vel[p] = v;
      s_par[p] = np;
      if (a.param_trace && cta == 0) a.param_trace[(size_t)s * BT_P + p] = np;
    }
    __syncthreads();
  }

  // Mirror the update to every executor replica (engine.py:313-315).
  if (cta == 0) {
    for (int x = 0; x < a.X; ++x) {
      double* rx = a.replicas + (size_t)x * 2 * BT_P;
      for (int i = tid; i < BT_P; i += T) {
        rx[i] = s_par[i];
        rx[BT_P + i] = s_vel[i];
      }
    }
  }
}

size_t mlp_smem_bytes(int nrows) {
  return sizeof(double) * ((size_t)3 * PAD_P + (size_t)nrows * (BT_INPUT_DIM + 1 + 4 * BT_HIDDEN + 3));
}

int mlp_launch(const bt_mlp_args& a, cudaStream_t stream) {
  const int grid = (a.E + a.est_per_cta - 1) / a.est_per_cta;
  const size_t smem = mlp_smem_bytes(a.est_per_cta * a.B);
  static bool attr_set = false;
  if (!attr_set) {
    if (cudaFuncSetAttribute(mlp_step_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024) !=
        cudaSuccess)
      return ERR_CUDA;
    attr_set = true;
  }
  cudaError_t err;
  if (grid > 1 && a.fuse_reduce) {
    if (cudaMemsetAsync(a.bar, 0, sizeof(uint32_t), stream) != cudaSuccess) return ERR_CUDA;
    void* params[] = {(void*)&a};
    err = cudaLaunchCooperativeKernel((const void*)mlp_step_kernel, dim3(grid), dim3(MLP_THREADS), params, smem,
                                      stream);
  } else {
    mlp_step_kernel<<<grid, MLP_THREADS, smem, stream>>>(a);
    err = cudaGetLastError();
  }
  return err == cudaSuccess ? OK : ERR_CUDA;
}

}  // namespace bt
