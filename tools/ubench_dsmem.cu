// DSMEM exchange microbenchmark: one cluster of G CTAs; every iteration each
// CTA delivers NP doubles to every CTA (all-to-all of the gradient slots) and
// waits for its own arrivals.  Variants: 0 = st.async f64 per (thread, peer),
// 1 = st.async v2.f64, 2 = cp.async.bulk smem->peer smem (one thread per peer),
// 3 = st.async to ONE peer only (latency floor), 4 = barrier.cluster only.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/ubench_dsmem tools/ubench_dsmem.cu
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

constexpr int NP = 168;  // padded slot (161 used)
__device__ __forceinline__ uint32_t su32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ uint32_t mapa(uint32_t a, int r) {
  uint32_t o; asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(o) : "r"(a), "r"(r)); return o; }
__device__ __forceinline__ bool try_wait(uint32_t bar, uint32_t ph) {
  uint32_t ok;
  asm volatile("{\n\t.reg .pred p;\n\tmbarrier.try_wait.parity.acquire.cluster.shared::cta.b64 p, [%1], %2;\n\tselp.u32 %0,1,0,p;\n\t}"
               : "=r"(ok) : "r"(bar), "r"(ph) : "memory");
  return ok; }
__device__ __forceinline__ bool try_wait_cta(uint32_t bar, uint32_t ph) {
  uint32_t ok;
  asm volatile("{\n\t.reg .pred p;\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\tselp.u32 %0,1,0,p;\n\t}"
               : "=r"(ok) : "r"(bar), "r"(ph) : "memory");
  return ok; }

template <int V>
__global__ void kern(int iters, int G, long long* out, int cta_scope) {
  extern __shared__ __align__(16) double sm[];  // [2][G][NP] slots + [NP] local
  __shared__ __align__(8) uint64_t bar[2];
  const int tid = threadIdx.x, cta = blockIdx.x;
  double* local = sm + 2 * G * NP;
  if (tid == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su32(&bar[0])));
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su32(&bar[1])));
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
  uint32_t peer[8], pbar[8];
  for (int r = 0; r < G; ++r) { peer[r] = mapa(su32(sm), r); pbar[r] = mapa(su32(&bar[0]), r); }
  uint32_t phases = 0;
  double val = tid * 1.0;
  long long t0 = clock64();
  for (int it = 0; it < iters; ++it) {
    const int par = it & 1;
    if (V == 4) {
      asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
      __syncthreads();
      continue;
    }
    uint32_t expect = V == 3 ? 161 * 8 : (uint32_t)G * (V == 2 ? NP : 161) * 8;
    if (V == 3) expect = (uint32_t)161 * 8;  // one sender (cta-1) per receiver
    if (tid == 0) asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(su32(&bar[par])), "r"(expect) : "memory");
    const uint32_t off = (uint32_t)(((par * G + cta) * NP) * 8);
    if (V == 0 && tid < 161) {
      for (int r = 0; r < G; ++r)
        asm volatile("st.async.shared::cluster.mbarrier::complete_tx::bytes.f64 [%0], %1, [%2];" ::"r"(peer[r] + off + tid * 8), "d"(val), "r"(pbar[r] + par * 8) : "memory");
    } else if (V == 1 && tid < 81) {
      const int p = 2 * tid;
      for (int r = 0; r < G; ++r) {
        if (p + 1 < 161)
          asm volatile("st.async.shared::cluster.mbarrier::complete_tx::bytes.v2.f64 [%0], {%1, %2}, [%3];" ::"r"(peer[r] + off + p * 8), "d"(val), "d"(val), "r"(pbar[r] + par * 8) : "memory");
        else
          asm volatile("st.async.shared::cluster.mbarrier::complete_tx::bytes.f64 [%0], %1, [%2];" ::"r"(peer[r] + off + p * 8), "d"(val), "r"(pbar[r] + par * 8) : "memory");
      }
    } else if (V == 2) {
      if (tid < 161) local[tid] = val;
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
      __syncthreads();
      if (tid < G)
        asm volatile("cp.async.bulk.shared::cluster.shared::cta.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(peer[tid] + off), "r"(su32(local)), "r"(NP * 8), "r"(pbar[tid] + par * 8) : "memory");
    } else if (V == 3 && tid < 161) {
      const int r = (cta + 1) % G;
      asm volatile("st.async.shared::cluster.mbarrier::complete_tx::bytes.f64 [%0], %1, [%2];" ::"r"(peer[r] + off + tid * 8), "d"(val), "r"(pbar[r] + par * 8) : "memory");
    }
    const uint32_t b = su32(&bar[par]), want = (phases >> par) & 1;
    if (cta_scope) { while (!try_wait_cta(b, want)) {} } else { while (!try_wait(b, want)) {} }
    phases ^= 1u << par;
    val += sm[(par * G + (tid % G)) * NP + (tid % 161)];
    __syncthreads();
  }
  long long t1 = clock64();
  asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
  if (tid == 0) out[cta] = (t1 - t0) / iters;
  if (val == 12345.0) out[G] = 1;
}

int main() {
  long long* d; cudaMalloc(&d, 64 * 8);
  long long h[16];
  const char* names[] = {"st.async f64 x G", "st.async v2 x G", "bulk copy x G", "st.async 1 peer", "cluster barrier"};
  for (int cta_scope = 0; cta_scope < 2; ++cta_scope)
  for (int G : {4, 8}) {
    for (int V = 0; V < 5; ++V) {
      size_t smem = (2 * G * NP + NP) * 8;
      cudaLaunchConfig_t cfg = {}; cfg.gridDim = dim3(G); cfg.blockDim = dim3(192); cfg.dynamicSmemBytes = smem;
      cudaLaunchAttribute at[1]; at[0].id = cudaLaunchAttributeClusterDimension; at[0].val.clusterDim.x = G;
      at[0].val.clusterDim.y = 1; at[0].val.clusterDim.z = 1; cfg.attrs = at; cfg.numAttrs = 1;
      cudaError_t e;
      for (int rep = 0; rep < 2; ++rep) {
        switch (V) {
          case 0: e = cudaLaunchKernelEx(&cfg, kern<0>, 2000, G, d, cta_scope); break;
          case 1: e = cudaLaunchKernelEx(&cfg, kern<1>, 2000, G, d, cta_scope); break;
          case 2: e = cudaLaunchKernelEx(&cfg, kern<2>, 2000, G, d, cta_scope); break;
          case 3: e = cudaLaunchKernelEx(&cfg, kern<3>, 2000, G, d, cta_scope); break;
          default: e = cudaLaunchKernelEx(&cfg, kern<4>, 2000, G, d, cta_scope); break;
        }
        if (e != cudaSuccess) { printf("launch err %s\n", cudaGetErrorString(e)); return 1; }
        e = cudaDeviceSynchronize();
        if (e != cudaSuccess) { printf("run err %s\n", cudaGetErrorString(e)); return 1; }
      }
      cudaMemcpy(h, d, G * 8, cudaMemcpyDeviceToHost);
      long long mx = 0; for (int i = 0; i < G; ++i) mx = h[i] > mx ? h[i] : mx;
      printf("G=%d %-20s wait=%s : %lld cycles/iter\n", G, names[V], cta_scope ? "cta" : "cluster", mx);
    }
  }
  return 0;
}
