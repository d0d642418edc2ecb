// Probe of the TMA im2col mode (cuTensorMapEncodeIm2col + cp.async.bulk.tensor.4d...im2col) on sm_100a:
// loads one 32-pixel x 64-channel column for given (c, w, h, n) coordinates and (kw, kh) offsets and
// dumps it, to pin the coordinate convention against an explicit im2col.
//   nvcc -gencode arch=compute_100a,code=sm_100a -o tools/probe_im2col tools/probe_im2col.cu -lcuda
#include <cuda.h>
#include <cuda_bf16.h>
#include <cuda_runtime.h>
#include <cstdio>
#include <cstdint>
#include <vector>

__global__ void probe(const __grid_constant__ CUtensorMap map, int c, int w, int h, int n, int ow, int oh,
                      uint16_t* out) {
  __shared__ __align__(1024) uint16_t box[32 * 64];
  __shared__ __align__(8) uint64_t bar;
  const uint32_t sb = (uint32_t)__cvta_generic_to_shared(box), bb = (uint32_t)__cvta_generic_to_shared(&bar);
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(bb));
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bb), "r"(32 * 64 * 2) : "memory");
    asm volatile(
        "cp.async.bulk.tensor.4d.shared::cluster.global.im2col.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4, %5}], "
        "[%6], {%7, %8};" ::"r"(sb),
        "l"(&map), "r"(c), "r"(w), "r"(h), "r"(n), "r"(bb), "h"((uint16_t)ow), "h"((uint16_t)oh)
        : "memory");
    uint32_t ok = 0;
    while (!ok)
      asm volatile("{\n\t.reg .pred p;\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%1], 0;\n\tselp.u32 %0, 1, 0, p;\n\t}"
                   : "=r"(ok) : "r"(bb) : "memory");
  }
  __syncthreads();
  for (int i = threadIdx.x; i < 32 * 64; i += blockDim.x) out[i] = box[i];
}

int main() {
  const int N = 2, H = 6, W = 5, C = 64;
  std::vector<uint16_t> host(N * H * W * C);
  for (int n = 0; n < N; ++n)
    for (int h = 0; h < H; ++h)
      for (int w = 0; w < W; ++w)
        for (int c = 0; c < C; ++c) host[((n * H + h) * W + w) * C + c] = (uint16_t)(1 + n * 1000 + h * 100 + w * 10 + (c == 0 ? 0 : 5));
  uint16_t *x, *out;
  cudaMalloc(&x, host.size() * 2);
  cudaMalloc(&out, 32 * 64 * 2);
  cudaMemcpy(x, host.data(), host.size() * 2, cudaMemcpyHostToDevice);
  CUtensorMap map;
  const cuuint64_t dims[4] = {(cuuint64_t)C, (cuuint64_t)W, (cuuint64_t)H, (cuuint64_t)N};
  const cuuint64_t strides[3] = {(cuuint64_t)C * 2, (cuuint64_t)W * C * 2, (cuuint64_t)H * W * C * 2};
  const int lower[2] = {-1, -1}, upper[2] = {-1, -1};
  const cuuint32_t estr[4] = {1, 1, 1, 1};
  CUresult r = cuTensorMapEncodeIm2col(&map, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 4, x, dims, strides, lower, upper, 64, 32,
                                       estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                                       CU_TENSOR_MAP_L2_PROMOTION_NONE, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  printf("encode %d\n", (int)r);
  const int cases[][6] = {{0, -1, -1, 0, 0, 0}, {0, -1, -1, 0, 1, 1}, {0, 0, 0, 0, 0, 0}, {0, 0, 0, 0, 1, 1},
                          {0, 2, -1, 0, 0, 0}, {0, -1, -1, 1, 2, 2}};
  for (auto& cs : cases) {
    probe<<<1, 128>>>(map, cs[0], cs[1], cs[2], cs[3], cs[4], cs[5], out);
    cudaError_t e = cudaDeviceSynchronize();
    std::vector<uint16_t> o(32 * 64);
    cudaMemcpy(o.data(), out, o.size() * 2, cudaMemcpyDeviceToHost);
    printf("coords c=%d w=%d h=%d n=%d off(w,h)=(%d,%d) err=%d : ", cs[0], cs[1], cs[2], cs[3], cs[4], cs[5], (int)e);
    for (int p = 0; p < 32; ++p) printf("%d ", o[p * 64] ? o[p * 64] - 1 : -1);
    printf("| ch1 of px0: %d\n", o[1]);
  }
  return 0;
}
