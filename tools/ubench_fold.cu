// Latency of the stage-F sequence (8 LDS leaves -> Tree(2) fold -> /8 -> momentum SGD -> STS),
// loop-carried through the result so iterations serialise.  One warp; then 6 warps.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -fmad=false -o tools/ubench_fold tools/ubench_fold.cu
#include <cstdio>
#include <cuda_runtime.h>
__global__ void k(int iters, long long* out, double* sink) {
  __shared__ double col[8 * 168];
  __shared__ double par[168], vel[168];
  const int t = threadIdx.x % 161;
  for (int i = threadIdx.x; i < 8 * 168; i += blockDim.x) col[i] = i * 1e-3;
  for (int i = threadIdx.x; i < 168; i += blockDim.x) { par[i] = 0.5; vel[i] = 0.1; }
  __syncthreads();
  const int rot = (t * 7) & 7;
  double np = 0.0;
  long long t0 = clock64();
  for (int it = 0; it < iters; ++it) {
    const int bump = np == 12345.0 ? 1 : 0;  // loop-carried dependency
    double v[8];
#pragma unroll
    for (int kk = 0; kk < 8; ++kk) { int q = rot + kk + bump; q -= q >= 8 ? 8 : 0; v[kk] = col[q * 168 + t]; }
    double s = __dadd_rn(__dadd_rn(__dadd_rn(v[0], v[1]), __dadd_rn(v[2], v[3])), __dadd_rn(__dadd_rn(v[4], v[5]), __dadd_rn(v[6], v[7])));
    double g = __dmul_rn(s, 0.125);
    double vv = __dadd_rn(__dmul_rn(0.9, vel[t]), g);
    np = __dsub_rn(par[t], __dmul_rn(0.02, vv));
    vel[t] = vv;
    par[t] = np;
  }
  long long t1 = clock64();
  if (threadIdx.x == 0) out[0] = (t1 - t0) / iters;
  sink[threadIdx.x] = np;
}
__global__ void chain(int iters, long long* out, double* sink, double x) {
  double a = x;
  long long t0 = clock64();
  for (int i = 0; i < iters; ++i) a = __dadd_rn(a, 1e-9);
  long long t1 = clock64();
  if (threadIdx.x == 0) out[1] = (t1 - t0) / iters;
  sink[threadIdx.x] = a;
  __shared__ double sm[64];
  sm[threadIdx.x % 64] = a;
  __syncthreads();
  int idx = threadIdx.x % 64;
  t0 = clock64();
  for (int i = 0; i < iters; ++i) { double v = sm[idx]; idx = (int)(v * 0.0) + ((idx + 1) & 63); }
  t1 = clock64();
  if (threadIdx.x == 0) out[2] = (t1 - t0) / iters;
  sink[threadIdx.x + 1] = idx;
}
int main() {
  long long* d; double* s; cudaMalloc(&d, 64); cudaMalloc(&s, 4096);
  long long h[4];
  for (int th : {32, 192}) {
    k<<<1, th>>>(1000, d, s); k<<<1, th>>>(10000, d, s); cudaMemcpy(h, d, 8, cudaMemcpyDeviceToHost);
    printf("F sequence, %d threads: %lld cycles/iter\n", th, h[0]);
  }
  chain<<<1, 32>>>(10000, d, s, 1.0); chain<<<1, 32>>>(10000, d, s, 1.0); cudaMemcpy(h, d, 24, cudaMemcpyDeviceToHost);
  printf("dadd chain: %lld cycles/op; dependent LDS chain: %lld cycles/op\n", h[1], h[2]);
  return 0;
}
