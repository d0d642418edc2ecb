// bt_reduce.cu -- the deterministic fixed-order gradient reducer with the fused
// 1/E scale and momentum-SGD update (the north star's core product).
//
// Replaces the reference's functional allreduce (buckets.py:85-124) +
// sgd_step (model.py:199-213).  The fold order of every element is a pure
// function of (EST rank, fanin, rotation): CTA/thread/GPU counts never enter,
// so the same ESTs give the same bits on 1, 2, 4 or 8 GPUs.
//
// Two kernels:
//  * reduce_fast_kernel<T, E, F>: Sequential (F=0) or unrotated Tree(2)
//    (F=2, E a power of two) -- the HBM-bound production path.  16-byte
//    vector loads (float4 / double2) of E contribution streams, folded in
//    registers with a compile-time tree; streaming cache hints; grid sized to
//    the SM count.  HBM bytes per element: E*sizeof(T) (grads) + 4*sizeof(T)
//    (param, vel read + write).
//  * reduce_generic_kernel<T>: any E, any fanin, optional per-element
//    rotation (the reference's ring-chunk order under Tree, buckets.py:119-122),
//    pointer-table or strided contributions.  Used for parity variants.
#include "bt_common.cuh"
#include "bt_reduce.cuh"

namespace bt {

template <typename T> struct Vec16;
template <> struct Vec16<float> { using type = float4; static constexpr int W = 4; };
template <> struct Vec16<double> { using type = double2; static constexpr int W = 2; };

__device__ __forceinline__ float lane(const float4& v, int w) { return w == 0 ? v.x : w == 1 ? v.y : w == 2 ? v.z : v.w; }
__device__ __forceinline__ double lane(const double2& v, int w) { return w == 0 ? v.x : v.y; }
__device__ __forceinline__ void set_lane(float4& v, int w, float x) {
  if (w == 0) v.x = x; else if (w == 1) v.y = x; else if (w == 2) v.z = x; else v.w = x;
}
__device__ __forceinline__ void set_lane(double2& v, int w, double x) { if (w == 0) v.x = x; else v.y = x; }

__device__ __forceinline__ void flag_numeric(int32_t* flags, int64_t idx) {
  atomicCAS(flags + FLAG_STATUS, 0, (int)ERR_NUMERIC);
  atomicMin(flags + FLAG_DETAIL, (int)(idx < 0x7fffffff ? idx : 0x7fffffff));
}

template <typename T>
__device__ __forceinline__ T elem(const bt_reduce_args& a, int k, int64_t p) {
  const T* base = a.grads_ld > 0 ? (const T*)a.grads[0] + (size_t)k * a.grads_ld : (const T*)a.grads[k];
  return base[p];
}

// Adam for one element, every operation round-to-nearest in a fixed order (no contraction):
// m' = mu*m + (1-mu)*g; s' = b2*s + (1-b2)*(g*g); p' = p - lr*(m'*bc1) / (sqrt(s'*bc2) + eps)
template <typename T>
__device__ __forceinline__ void adam_elem(const bt_reduce_args& a, T g, T m, T s2, T p, T* mo, T* so, T* po) {
  using A = Arith<T>;
  const T b1 = (T)a.mu, b2 = (T)a.beta2;
  const T m1 = A::add(A::mul(b1, m), A::mul(A::sub((T)1, b1), g));
  const T s1 = A::add(A::mul(b2, s2), A::mul(A::sub((T)1, b2), A::mul(g, g)));
  const T den = A::add(sqrt(A::mul(s1, (T)a.bc2)), (T)a.eps);
  *mo = m1;
  *so = s1;
  *po = A::sub(p, A::mul((T)a.lr, A::div(A::mul(m1, (T)a.bc1), den)));
}

template <typename T>
__device__ __forceinline__ void update_elem(const bt_reduce_args& a, int64_t p, T g);

// Apply /E, finite check and the update for one element.
template <typename T>
__device__ __forceinline__ void finish_elem(const bt_reduce_args& a, int64_t p, T sum) {
  if (a.mode == BT_REDUCE_SUM_ONLY) {
    ((T*)a.param_out)[p] = sum;
    return;
  }
  const T g = Arith<T>::div(sum, (T)(a.divisor > 0 ? a.divisor : a.E));
  if (a.mode == BT_REDUCE_MEAN_ONLY || a.mode == BT_REDUCE_MEAN_CHECK) {
    if (a.mode == BT_REDUCE_MEAN_CHECK && !finite_v(g)) flag_numeric(a.flags, p);
    ((T*)a.param_out)[p] = g;
    return;
  }
  if (!finite_v(g)) flag_numeric(a.flags, p);
  update_elem<T>(a, p, g);
}

// The update of one element from its synchronized gradient g (momentum SGD or Adam) + replicas.
template <typename T>
__device__ __forceinline__ void update_elem(const bt_reduce_args& a, int64_t p, T g) {
  if (a.mode == BT_REDUCE_ADAM) {
    T m, s2, np;
    adam_elem<T>(a, g, ((const T*)a.vel)[p], ((const T*)a.vel2)[p], ((const T*)a.param)[p], &m, &s2, &np);
    ((T*)a.vel_out)[p] = m;
    ((T*)a.vel2_out)[p] = s2;
    ((T*)a.param_out)[p] = np;
    for (int r = 0; r < a.nout; ++r) {
      ((T*)a.extra_param_out[r])[p] = np;
      ((T*)a.extra_vel_out[r])[p] = m;
      ((T*)a.extra_vel2_out[r])[p] = s2;
    }
    return;
  }
  const T v = Arith<T>::add(Arith<T>::mul((T)a.mu, ((const T*)a.vel)[p]), g);
  const T np = Arith<T>::sub(((const T*)a.param)[p], Arith<T>::mul((T)a.lr, v));
  ((T*)a.vel_out)[p] = v;
  ((T*)a.param_out)[p] = np;
  for (int r = 0; r < a.nout; ++r) {
    ((T*)a.extra_param_out[r])[p] = np;
    ((T*)a.extra_vel_out[r])[p] = v;
  }
}

template <typename T>
__global__ void __launch_bounds__(256) reduce_generic_kernel(const __grid_constant__ bt_reduce_args a) {
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t p = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; p < a.n; p += stride) {
    const int start = a.rot ? a.rot[p] : 0;
    StreamFold<T, 24> f;
    f.init(a.fanin);
    for (int k = 0; k < a.E; ++k) {
      int src = start + k;
      if (src >= a.E) src -= a.E;
      f.push(elem<T>(a, src, p));
    }
    finish_elem<T>(a, p, f.finish());
  }
}

template <typename V>
__device__ __forceinline__ V ld_stream(const V* p) { return __ldcs(p); }
template <typename V>
__device__ __forceinline__ void st_stream(V* p, const V& v) { __stcs(p, v); }

template <typename T>
__device__ __forceinline__ void update_vec(const bt_reduce_args& a, int64_t i, const typename Vec16<T>::type& g);

// E in {1,2,4,...,64}; F == 0 (Sequential) or F == 2 (unrotated Tree(2)).
template <typename T, int E, int F>
__global__ void __launch_bounds__(256) reduce_fast_kernel(const __grid_constant__ bt_reduce_args a) {
  using V = typename Vec16<T>::type;
  constexpr int W = Vec16<T>::W;
  constexpr int C = E < 16 ? E : 16;  // contributions loaded per chunk
  constexpr int NC = E / C;           // chunks (power-of-two E => exact)
  const int64_t nv = a.n / W;
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  const T invE_dummy = (T)0;  // (division below is a true /E, never *1/E)
  (void)invE_dummy;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < nv; i += stride) {
    T sum[W];
    T part[NC > 1 ? NC : 1][W];
#pragma unroll
    for (int c = 0; c < NC; ++c) {
      V buf[C];
#pragma unroll
      for (int k = 0; k < C; ++k) buf[k] = ld_stream((const V*)a.grads[c * C + k] + i);
#pragma unroll
      for (int w = 0; w < W; ++w) {
        if (F == 0) {  // strict left fold over ranks, continued across chunks
          T acc = c == 0 ? lane(buf[0], w) : Arith<T>::add(sum[w], lane(buf[0], w));
#pragma unroll
          for (int k = 1; k < C; ++k) acc = Arith<T>::add(acc, lane(buf[k], w));
          sum[w] = acc;
        } else {  // complete binary tree: chunk subtrees, then the top levels
          T v[C];
#pragma unroll
          for (int k = 0; k < C; ++k) v[k] = lane(buf[k], w);
          part[c][w] = TreeLevel<C, 2>::run(v);
        }
      }
    }
    if (F != 0) {
#pragma unroll
      for (int w = 0; w < W; ++w) {
        T v[NC];
#pragma unroll
        for (int c = 0; c < NC; ++c) v[c] = part[c][w];
        sum[w] = TreeLevel<NC, 2>::run(v);
      }
    }
    if (a.mode == BT_REDUCE_SUM_ONLY) {  // per-GPU subtree partial (hierarchical path)
      V sv;
#pragma unroll
      for (int w = 0; w < W; ++w) set_lane(sv, w, sum[w]);
      st_stream((V*)a.param_out + i, sv);
      continue;
    }
    V g;
    bool fin = true;
    const T div = (T)(a.divisor > 0 ? a.divisor : E);
#pragma unroll
    for (int w = 0; w < W; ++w) {
      const T gw = Arith<T>::div(sum[w], div);
      set_lane(g, w, gw);
      fin = fin && finite_v(gw);
    }
    if (a.mode == BT_REDUCE_MEAN_ONLY || a.mode == BT_REDUCE_MEAN_CHECK) {
      if (a.mode == BT_REDUCE_MEAN_CHECK && !fin) flag_numeric(a.flags, i * W);
      st_stream((V*)a.param_out + i, g);
      continue;
    }
    if (!fin) flag_numeric(a.flags, i * W);
    update_vec<T>(a, i, g);
  }
  // scalar tail (n % W elements)
  if (blockIdx.x == 0) {
    for (int64_t p = nv * W + threadIdx.x; p < a.n; p += blockDim.x) {
      T acc = ((const T*)a.grads[0])[p];
      if (F == 0) {
        for (int k = 1; k < E; ++k) acc = Arith<T>::add(acc, ((const T*)a.grads[k])[p]);
      } else {
        T v[E];
#pragma unroll
        for (int k = 0; k < E; ++k) v[k] = ((const T*)a.grads[k])[p];
        acc = TreeLevel<E, 2>::run(v);
      }
      finish_elem<T>(a, p, acc);
    }
  }
}

// The update of 16 bytes of elements from their synchronized gradients g, + replicas.
template <typename T>
__device__ __forceinline__ void update_vec(const bt_reduce_args& a, int64_t i, const typename Vec16<T>::type& g) {
  using V = typename Vec16<T>::type;
  constexpr int W = Vec16<T>::W;
  {
    const V pv = ld_stream((const V*)a.param + i);
    const V vv = ld_stream((const V*)a.vel + i);
    V nv_, np_;
    if (a.mode == BT_REDUCE_ADAM) {
      const V sv = ld_stream((const V*)a.vel2 + i);
      V ns_;
#pragma unroll
      for (int w = 0; w < W; ++w) {
        T m, s2, np;
        adam_elem<T>(a, lane(g, w), lane(vv, w), lane(sv, w), lane(pv, w), &m, &s2, &np);
        set_lane(nv_, w, m);
        set_lane(ns_, w, s2);
        set_lane(np_, w, np);
      }
      st_stream((V*)a.vel_out + i, nv_);
      st_stream((V*)a.vel2_out + i, ns_);
      st_stream((V*)a.param_out + i, np_);
      for (int r = 0; r < a.nout; ++r) {
        st_stream((V*)a.extra_param_out[r] + i, np_);
        st_stream((V*)a.extra_vel_out[r] + i, nv_);
        st_stream((V*)a.extra_vel2_out[r] + i, ns_);
      }
      return;
    }
#pragma unroll
    for (int w = 0; w < W; ++w) {
      const T v = Arith<T>::add(Arith<T>::mul((T)a.mu, lane(vv, w)), lane(g, w));
      set_lane(nv_, w, v);
      set_lane(np_, w, Arith<T>::sub(lane(pv, w), Arith<T>::mul((T)a.lr, v)));
    }
    st_stream((V*)a.vel_out + i, nv_);
    st_stream((V*)a.param_out + i, np_);
    for (int r = 0; r < a.nout; ++r) {
      st_stream((V*)a.extra_param_out[r] + i, np_);
      st_stream((V*)a.extra_vel_out[r] + i, nv_);
    }
  }
}

// Pass 2 of a guarded update: the update from the staged synchronized gradients, applied only
// when this update's status (and every other rank's published status) is clean.
__device__ __forceinline__ bool gate_open(const bt_reduce_args& a) {
  if (a.flags[FLAG_STATUS] != 0) return false;
  for (int i = 0; i < a.ngate; ++i)
    if (((volatile const int32_t*)a.gate)[i] != 0) return false;
  return true;
}

template <typename T, bool VEC>
__global__ void __launch_bounds__(256) reduce_apply_kernel(const __grid_constant__ bt_reduce_args a) {
  __shared__ int s_open;
  if (threadIdx.x == 0) {
    s_open = gate_open(a);
    if (!s_open && blockIdx.x == 0 && a.flags[FLAG_STATUS] == 0)
      atomicCAS(a.flags + FLAG_STATUS, 0, (int)ERR_NUMERIC);  // another rank's shard was not finite
  }
  __syncthreads();
  if (!s_open) return;
  using V = typename Vec16<T>::type;
  constexpr int W = Vec16<T>::W;
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  const int64_t t0 = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (VEC) {
    const int64_t nv = a.n / W;
    for (int64_t i = t0; i < nv; i += stride) update_vec<T>(a, i, ld_stream((const V*)a.stage + i));
    if (blockIdx.x == 0)
      for (int64_t p = nv * W + threadIdx.x; p < a.n; p += blockDim.x) update_elem<T>(a, p, ((const T*)a.stage)[p]);
  } else {
    for (int64_t p = t0; p < a.n; p += stride) update_elem<T>(a, p, ((const T*)a.stage)[p]);
  }
}

static int g_num_sms = 0;
static int num_sms() {
  if (g_num_sms == 0) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&g_num_sms, cudaDevAttrMultiProcessorCount, dev);
    if (g_num_sms <= 0) g_num_sms = 148;
  }
  return g_num_sms;
}

template <typename T, int E, int F>
static cudaError_t launch_fast(const bt_reduce_args& a, cudaStream_t s) {
  constexpr int W = Vec16<T>::W;
  const int64_t nv = (a.n + W - 1) / W;
  int64_t blocks = (nv + 255) / 256;
  const int64_t cap = (int64_t)num_sms() * 8;  // 8 x 256 threads resident per SM
  if (blocks > cap) blocks = cap;
  if (blocks < 1) blocks = 1;
  reduce_fast_kernel<T, E, F><<<(unsigned)blocks, 256, 0, s>>>(a);
  return cudaGetLastError();
}

template <typename T, int F>
static cudaError_t dispatch_fast_E(const bt_reduce_args& a, cudaStream_t s, bool* taken) {
  *taken = true;
  switch (a.E) {
    case 1: return launch_fast<T, 1, F>(a, s);
    case 2: return launch_fast<T, 2, F>(a, s);
    case 4: return launch_fast<T, 4, F>(a, s);
    case 8: return launch_fast<T, 8, F>(a, s);
    case 16: return launch_fast<T, 16, F>(a, s);
    case 32: return launch_fast<T, 32, F>(a, s);
    case 64: return launch_fast<T, 64, F>(a, s);
    default: *taken = false; return cudaSuccess;
  }
}

static bool aligned16(const void* p) { return ((uintptr_t)p & 15u) == 0; }

template <typename T>
static cudaError_t reduce_launch_t(const bt_reduce_args& a, cudaStream_t s) {
  bool fast_ok = a.rot == nullptr && a.grads_ld == 0 && (a.fanin == 0 || a.fanin == 2);
  if (fast_ok) {
    for (int k = 0; k < a.E; ++k) fast_ok = fast_ok && aligned16(a.grads[k]);
    fast_ok = fast_ok && aligned16(a.param_out);
    if (a.mode == BT_REDUCE_UPDATE || a.mode == BT_REDUCE_ADAM) {  // (SUM_ONLY / MEAN_ONLY only write param_out)
      fast_ok = fast_ok && aligned16(a.param) && aligned16(a.vel) && aligned16(a.vel_out);
      for (int r = 0; r < a.nout; ++r) fast_ok = fast_ok && aligned16(a.extra_param_out[r]) && aligned16(a.extra_vel_out[r]);
      if (a.mode == BT_REDUCE_ADAM) {
        fast_ok = fast_ok && aligned16(a.vel2) && aligned16(a.vel2_out);
        for (int r = 0; r < a.nout; ++r) fast_ok = fast_ok && aligned16(a.extra_vel2_out[r]);
      }
    }
  }
  if (fast_ok) {
    bool taken = false;
    cudaError_t e = a.fanin == 0 ? dispatch_fast_E<T, 0>(a, s, &taken) : dispatch_fast_E<T, 2>(a, s, &taken);
    if (taken) return e;
  }
  int64_t blocks = (a.n + 255) / 256;
  const int64_t cap = (int64_t)num_sms() * 8;
  if (blocks > cap) blocks = cap;
  if (blocks < 1) blocks = 1;
  reduce_generic_kernel<T><<<(unsigned)blocks, 256, 0, s>>>(a);
  return cudaGetLastError();
}

template <typename T>
static cudaError_t apply_launch_t(const bt_reduce_args& a, cudaStream_t s) {
  bool vec = aligned16(a.stage) && aligned16(a.param) && aligned16(a.vel) && aligned16(a.param_out) &&
             aligned16(a.vel_out);
  for (int r = 0; r < a.nout; ++r) vec = vec && aligned16(a.extra_param_out[r]) && aligned16(a.extra_vel_out[r]);
  if (a.mode == BT_REDUCE_ADAM) {
    vec = vec && aligned16(a.vel2) && aligned16(a.vel2_out);
    for (int r = 0; r < a.nout; ++r) vec = vec && aligned16(a.extra_vel2_out[r]);
  }
  int64_t blocks = (a.n / (vec ? Vec16<T>::W : 1) + 255) / 256;
  const int64_t cap = (int64_t)num_sms() * 8;
  if (blocks > cap) blocks = cap;
  if (blocks < 1) blocks = 1;
  if (vec) reduce_apply_kernel<T, true><<<(unsigned)blocks, 256, 0, s>>>(a);
  else reduce_apply_kernel<T, false><<<(unsigned)blocks, 256, 0, s>>>(a);
  return cudaGetLastError();
}

int reduce_launch(const bt_reduce_args& a, cudaStream_t s) {
  if (a.n == 0) return OK;
  const bool f64 = a.dtype == BT_DTYPE_F64;
  if (a.mode == BT_REDUCE_APPLY_SGD || a.mode == BT_REDUCE_APPLY_ADAM) {  // pass 2 of a multi-rank guard
    bt_reduce_args p2 = a;
    p2.mode = a.mode == BT_REDUCE_APPLY_ADAM ? BT_REDUCE_ADAM : BT_REDUCE_UPDATE;
    const cudaError_t e = f64 ? apply_launch_t<double>(p2, s) : apply_launch_t<float>(p2, s);
    return e == cudaSuccess ? OK : ERR_CUDA;
  }
  if (a.stage && (a.mode == BT_REDUCE_UPDATE || a.mode == BT_REDUCE_ADAM)) {  // guarded: check, then apply
    bt_reduce_args p1 = a;
    p1.mode = BT_REDUCE_MEAN_CHECK;
    p1.param_out = a.stage;
    p1.nout = 0;
    cudaError_t e = f64 ? reduce_launch_t<double>(p1, s) : reduce_launch_t<float>(p1, s);
    if (e != cudaSuccess) return ERR_CUDA;
    e = f64 ? apply_launch_t<double>(a, s) : apply_launch_t<float>(a, s);
    return e == cudaSuccess ? OK : ERR_CUDA;
  }
  const cudaError_t e = f64 ? reduce_launch_t<double>(a, s) : reduce_launch_t<float>(a, s);
  return e == cudaSuccess ? OK : ERR_CUDA;
}

// ---------------------------------------------------------- small seams
// reduce_sum(values, variant) for one list (reduction.py:51-62).
__global__ void reduce_sum_kernel(const double* v, int64_t n, int fanin, double* out) {
  if (threadIdx.x != 0 || blockIdx.x != 0) return;
  StreamFold<double, 64> f;
  f.init(fanin);
  for (int64_t i = 0; i < n; ++i) f.push(v[i]);
  *out = f.finish();
}

int reduce_sum_launch(const double* v, int64_t n, int fanin, double* out, cudaStream_t s) {
  reduce_sum_kernel<<<1, 32, 0, s>>>(v, n, fanin, out);
  return cudaGetLastError() == cudaSuccess ? OK : ERR_CUDA;
}

// sgd_step (model.py:199-213), out of place; NUMERIC flag + first bad index.
__global__ void sgd_kernel(const double* p, const double* v, const double* g, int64_t n, double lr, double mu,
                           double* po, double* vo, int32_t* flags) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    const double gi = g[i];
    if (!finite_d(gi)) flag_numeric(flags, i);
    const double vi = dadd(dmul(mu, v[i]), gi);
    vo[i] = vi;
    po[i] = dsub(p[i], dmul(lr, vi));
  }
}

int sgd_launch(const double* p, const double* v, const double* g, int64_t n, double lr, double mu, double* po,
               double* vo, int32_t* flags, cudaStream_t s) {
  int64_t blocks = (n + 255) / 256;
  if (blocks > 4096) blocks = 4096;
  if (blocks < 1) blocks = 1;
  sgd_kernel<<<(unsigned)blocks, 256, 0, s>>>(p, v, g, n, lr, mu, po, vo, flags);
  return cudaGetLastError() == cudaSuccess ? OK : ERR_CUDA;
}

}  // namespace bt
