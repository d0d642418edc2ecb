// packed f32x2 add/mul/fma vs the scalar round-to-nearest forms on random operands
#include <cstdio>
#include <cstdint>
#include "../paper_2208_14228_b200/csrc/bt_ffn.cuh"
using namespace bt::ffn;
__global__ void k(const float* x, int n, unsigned* bad) {
  int i = 4 * (blockIdx.x * blockDim.x + threadIdx.x);
  if (i + 3 >= n) return;
  float a = x[i], b = x[i + 1], c = x[i + 2], d = x[i + 3];
  float2 A = upk2(add2(pk2(a, b), pk2(c, d))), M = upk2(mul2(pk2(a, b), pk2(c, d))),
         F = upk2(fma2(pk2(a, b), pk2(c, d), pk2(b, a))), S = upk2(sub2(pk2(a, b), pk2(c, d)));
  if (__float_as_uint(A.x) != __float_as_uint(__fadd_rn(a, c)) || __float_as_uint(A.y) != __float_as_uint(__fadd_rn(b, d))) atomicAdd(bad, 1u);
  if (__float_as_uint(M.x) != __float_as_uint(__fmul_rn(a, c)) || __float_as_uint(M.y) != __float_as_uint(__fmul_rn(b, d))) atomicAdd(bad + 1, 1u);
  if (__float_as_uint(F.x) != __float_as_uint(__fmaf_rn(a, c, b)) || __float_as_uint(F.y) != __float_as_uint(__fmaf_rn(b, d, a))) atomicAdd(bad + 2, 1u);
  if (__float_as_uint(S.x) != __float_as_uint(__fsub_rn(a, c)) || __float_as_uint(S.y) != __float_as_uint(__fsub_rn(b, d))) atomicAdd(bad + 3, 1u);
  // fma with a negated product operand, the way gelu_and_grad writes it
  float2 G = upk2(fma2(sub2(pk2(c, d), pk2(1.f, 1.f)), pk2(a, b), pk2(1.f, 1.f)));
  if (__float_as_uint(G.x) != __float_as_uint(__fmaf_rn(-__fsub_rn(1.f, c), a, 1.f))) atomicAdd(bad + 4, 1u);
}
int main() {
  const int n = 1 << 24;
  float* h = (float*)malloc(n * 4);
  uint64_t s = 7;
  for (int i = 0; i < n; ++i) { s = s * 6364136223846793005ull + 1442695040888963407ull; h[i] = ((int)(s >> 40) - (1 << 23)) / (float)(1 << 22); }
  float* x; unsigned* bad;
  cudaMalloc(&x, n * 4); cudaMalloc(&bad, 20); cudaMemset(bad, 0, 20);
  cudaMemcpy(x, h, n * 4, cudaMemcpyHostToDevice);
  k<<<n / 1024, 256>>>(x, n, bad);
  unsigned b[5];
  cudaMemcpy(b, bad, 20, cudaMemcpyDeviceToHost);
  printf("mismatches of %d: add2 %u mul2 %u fma2 %u sub2 %u negfma %u\n", n / 4, b[0], b[1], b[2], b[3], b[4]);
}
