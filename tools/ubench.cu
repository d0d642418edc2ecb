// Latency micro-benchmarks on the B200 for the fp64 ops the step kernel chains.
#include <cstdio>
#include "../paper_2208_14228_b200/csrc/bt_libm.cuh"

__global__ void k(double* out, long long* cyc, double x0, int n) {
  __shared__ double sm[1024];
  double x = x0 + threadIdx.x * 1e-9, y = 1.0000001;
  long long t0, t1;
  // dadd chain
  t0 = clock64(); for (int i = 0; i < n; ++i) x = bt::dadd(x, y); t1 = clock64(); if (threadIdx.x == 0) cyc[0] = (t1 - t0);
  t0 = clock64(); for (int i = 0; i < n; ++i) x = bt::dmul(x, y); t1 = clock64(); if (threadIdx.x == 0) cyc[1] = (t1 - t0);
  t0 = clock64(); for (int i = 0; i < n; ++i) x = bt::ddiv(x, y); t1 = clock64(); if (threadIdx.x == 0) cyc[2] = (t1 - t0);
  double z = 0.3;
  t0 = clock64(); for (int i = 0; i < n; ++i) z = bt::glibc_tanh(z + 0.5); t1 = clock64(); if (threadIdx.x == 0) cyc[3] = (t1 - t0);
  sm[threadIdx.x] = x;
  __syncthreads();
  t0 = clock64(); for (int i = 0; i < n; ++i) { double v = sm[(threadIdx.x + i) & 1023]; sm[(threadIdx.x + i + 1) & 1023] = bt::dadd(v, 1.0); } t1 = clock64(); if (threadIdx.x == 0) cyc[4] = (t1 - t0);
  t0 = clock64(); for (int i = 0; i < n; ++i) __syncthreads(); t1 = clock64(); if (threadIdx.x == 0) cyc[5] = (t1 - t0);
  t0 = clock64(); for (int i = 0; i < n; ++i) x = bt::dfma(x, y, 1e-9); t1 = clock64(); if (threadIdx.x == 0) cyc[6] = (t1 - t0);
  float f = x; t0 = clock64(); for (int i = 0; i < n; ++i) f = __fadd_rn(f, 1.0f); t1 = clock64(); if (threadIdx.x == 0) cyc[7] = (t1 - t0);
  out[threadIdx.x] = x + z + f + sm[threadIdx.x];
}
int main() {
  double* out; long long* cyc; cudaMalloc(&out, 8192); cudaMallocManaged(&cyc, 64);
  const char* names[] = {"dadd", "dmul", "ddiv", "glibc_tanh", "lds-dadd-sts", "syncthreads(512)", "dfma", "fadd"};
  for (int threads : {32, 512}) {
    k<<<1, threads>>>(out, cyc, 0.5, 1000); cudaDeviceSynchronize();
    k<<<1, threads>>>(out, cyc, 0.5, 1000); cudaDeviceSynchronize();
    printf("threads=%d:", threads);
    for (int i = 0; i < 8; ++i) printf("  %s %.1f", names[i], cyc[i] / 1000.0);
    printf("  (cycles/op)\n");
  }
  return 0;
}
