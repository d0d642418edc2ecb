// mma.sync m16n8k16 bf16 throughput on sm_100a (does the legacy warp-level tensor path bound attention?)
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/ubench_mma tools/ubench_mma.cu && tools/ubench_mma
#include <cstdio>
#include <cuda_runtime.h>
#include <stdint.h>
__global__ void k(float* out, int iters) {
  float c[8][4] = {};
  uint32_t a[4] = {threadIdx.x, threadIdx.x * 3u, threadIdx.x ^ 5u, 7u};
  uint32_t b0 = threadIdx.x * 11u, b1 = 13u;
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int j = 0; j < 8; ++j)
      asm volatile("mma.sync.aligned.m16n8k16.row.col.f32.bf16.bf16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, {%0,%1,%2,%3};"
                   : "+f"(c[j][0]), "+f"(c[j][1]), "+f"(c[j][2]), "+f"(c[j][3])
                   : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b0), "r"(b1));
  }
  float s = 0;
  for (int j = 0; j < 8; ++j) s += c[j][0] + c[j][1] + c[j][2] + c[j][3];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}
int main() {
  float* out;
  cudaMalloc(&out, 148 * 8 * 1024 * 4);
  for (int threads : {128, 256, 512, 1024}) {
    int iters = 4096, blocks = 148 * 2;
    k<<<blocks, threads>>>(out, 16);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    cudaEventRecord(e0);
    k<<<blocks, threads>>>(out, iters);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    double flops = 2.0 * 16 * 8 * 16 * 8.0 * iters * (threads / 32) * blocks;
    printf("threads/CTA %4d x %d CTAs: %.1f TF/s (mma.sync m16n8k16 bf16)\n", threads, blocks, flops / ms / 1e9);
  }
  return 0;
}
