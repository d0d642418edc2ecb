// Latency of the step kernel's building blocks on B200 (single warp, dependent chains).
#include <cstdio>
#include <cooperative_groups.h>
#include "../paper_2208_14228_b200/csrc/bt_libm.cuh"
namespace cg = cooperative_groups;
__global__ void k(double* out, long long* cyc, double x0, int n) {
  double z = x0 + threadIdx.x * 1e-3;
  long long t0 = clock64();
  for (int i = 0; i < n; ++i) z = bt::glibc_tanh_simt(z + 0.75);
  long long t1 = clock64();
  if (threadIdx.x == 0) cyc[0] = t1 - t0;
  double y = z;
  t0 = clock64();
  for (int i = 0; i < n; ++i) y = bt::ddiv(y, 1.0000001);
  t1 = clock64();
  if (threadIdx.x == 0) cyc[1] = t1 - t0;
  uint64_t s = (uint64_t)(y * 1e6);
  t0 = clock64();
  for (int i = 0; i < n; ++i) s = bt::mix64(s + i);
  t1 = clock64();
  if (threadIdx.x == 0) cyc[2] = t1 - t0;
  double w = bt::unit_float(s);
  t0 = clock64();
  for (int i = 0; i < n; ++i) w = (double)(int)bt::dadd(bt::dmul(1.4426950408889634, w), 0.5);
  t1 = clock64();
  if (threadIdx.x == 0) cyc[3] = t1 - t0;
  out[threadIdx.x] = z + y + w + (double)s;
}
__global__ void __cluster_dims__(8, 1, 1) kc(double* out, long long* cyc, int n) {
  __shared__ double buf[256];
  buf[threadIdx.x] = threadIdx.x;
  cg::this_cluster().sync();
  long long t0 = clock64();
  for (int i = 0; i < n; ++i) asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
  long long t1 = clock64();
  if (threadIdx.x == 0 && blockIdx.x == 0) cyc[4] = t1 - t0;
  t0 = clock64();
  for (int i = 0; i < n; ++i) __syncthreads();
  t1 = clock64();
  if (threadIdx.x == 0 && blockIdx.x == 0) cyc[5] = t1 - t0;
  const double* peer = cg::this_cluster().map_shared_rank(buf, (blockIdx.x + 1) % 8);
  double acc = 0; int idx = threadIdx.x;
  t0 = clock64();
  for (int i = 0; i < n; ++i) { acc += peer[idx]; idx = ((int)acc + i) & 255; }
  t1 = clock64();
  if (threadIdx.x == 0 && blockIdx.x == 0) cyc[6] = t1 - t0;
  cg::this_cluster().sync();
  out[threadIdx.x] = acc;
}
int main() {
  double* out; long long* cyc; cudaMalloc(&out, 8192); cudaMallocManaged(&cyc, 128);
  for (int rep = 0; rep < 2; ++rep) {
    k<<<1, 32>>>(out, cyc, 0.5, 1000); kc<<<8, 192>>>(out, cyc, 1000); cudaDeviceSynchronize();
  }
  printf("tanh_simt %.1f  ddiv %.1f  mix64 %.1f  cvt-chain %.1f  cluster_barrier(8x192) %.1f  syncthreads(192) %.1f  dsmem_load %.1f cycles/op\n",
         cyc[0] / 1000.0, cyc[1] / 1000.0, cyc[2] / 1000.0, cyc[3] / 1000.0, cyc[4] / 1000.0, cyc[5] / 1000.0, cyc[6] / 1000.0);
  return 0;
}
