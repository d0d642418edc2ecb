// Stage-B building blocks in isolation (one warp): where do the cycles go?
#include <cstdio>
#include "../paper_2208_14228_b200/csrc/bt_libm.cuh"

__global__ void k(const double* gdata, long long* cyc, int n, int use_generic) {
  __shared__ double s_data[512 * 9];
  __shared__ double s_par[168];
  __shared__ int s_idx[64];
  __shared__ double s_x[64 * 8];
  for (int i = threadIdx.x; i < 512 * 9; i += blockDim.x) s_data[i] = gdata[i];
  for (int i = threadIdx.x; i < 168; i += blockDim.x) s_par[i] = 0.01 * i;
  for (int i = threadIdx.x; i < 64; i += blockDim.x) s_idx[i] = (i * 37) % 512;
  __syncthreads();
  const double* data = use_generic ? (const double*)((uintptr_t)s_data | 0) : s_data;
  if (use_generic == 2) data = gdata;
  if (use_generic == 3) data = s_data;
  const int j = threadIdx.x & 15, row = threadIdx.x >> 4;
  double accsum = 0;
  long long ta = 0, tb = 0, tc = 0;
  for (int s = 0; s < n; ++s) {
    long long t0 = clock64();
    const int idx = s_idx[(row + s) & 63];
    const double* src = data + (size_t)idx * 9;
    double x[8];
#pragma unroll
    for (int i = 0; i < 8; ++i) x[i] = bt::dadd(src[i], 0.001 * s);
    if (use_generic == 3) {
#pragma unroll
      for (int i = 0; i < 8; ++i)
        if (j == i) s_x[row * 8 + i] = x[i];
    }
    long long t1 = clock64();
    double acc = bt::dmul(s_par[j], x[0]);
#pragma unroll
    for (int i = 1; i < 8; ++i) acc = bt::dadd(acc, bt::dmul(s_par[i * 16 + j], x[i]));
    const double pre = bt::dadd(acc, s_par[128 + j]);
    asm volatile("" ::"d"(pre));
    long long t2 = clock64();
    const double act = bt::glibc_tanh_simt(pre);
    asm volatile("" ::"d"(act));
    long long t3 = clock64();
    s_x[threadIdx.x] = act;
    accsum += act;
    ta += t1 - t0; tb += t2 - t1; tc += t3 - t2;
    __syncwarp();
  }
  if (threadIdx.x == 0) { cyc[0] = ta / n; cyc[1] = tb / n; cyc[2] = tc / n; }
  if (accsum == 12345.0) cyc[3] = 1;
}
int main() {
  double* g; long long* cyc; cudaMalloc(&g, 1024 * 9 * 8); cudaMemset(g, 0, 1024 * 72); cudaMallocManaged(&cyc, 64);
  for (int mode = 0; mode < 4; ++mode) {
    for (int r = 0; r < 2; ++r) { k<<<1, 32>>>(g, cyc, 200, mode); cudaDeviceSynchronize(); }
    printf("mode=%d (0 smem ptr, 1 generic-to-smem, 2 global): loads %lld  preact %lld  tanh %lld cycles\n", mode, cyc[0], cyc[1], cyc[2]);
  }
}
