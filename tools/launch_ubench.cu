// Host cost of kernel launches on this box: plain <<<>>>, cudaLaunchKernelEx with a cluster
// attribute, and cudaGraphLaunch of the same cluster launch (+ kernel-node param update).
// nvcc -gencode arch=compute_100a,code=sm_100a -O2 tools/launch_ubench.cu -o tools/launch_ubench [--cudart shared]
#include <chrono>
#include <cstdio>
#include <algorithm>
#include <vector>
#include <cuda_runtime.h>

struct Args { long long x[40]; };
__global__ void empty_k(const __grid_constant__ Args a, int* out) { if (threadIdx.x == 0 && a.x[0] == -1) *out = 1; }

template <class F>
static double med_us(F f, int n = 2000) {
  std::vector<double> t;
  for (int i = 0; i < n; ++i) {
    auto t0 = std::chrono::steady_clock::now();
    f();
    auto t1 = std::chrono::steady_clock::now();
    t.push_back(std::chrono::duration<double, std::micro>(t1 - t0).count());
  }
  std::sort(t.begin(), t.end());
  return t[t.size() / 2];
}

int main() {
  cudaStream_t s;
  cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking);
  int* out;
  cudaMalloc(&out, 4);
  Args a = {};
  cudaFuncSetAttribute(empty_k, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
  printf("plain     %.2f us\n", med_us([&] { empty_k<<<8, 192, 0, s>>>(a, out); }));
  cudaStreamSynchronize(s);
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(8);
  cfg.blockDim = dim3(192);
  cfg.dynamicSmemBytes = 200 * 1024;
  cfg.stream = s;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = 8;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  printf("cluster   %.2f us\n", med_us([&] { cudaLaunchKernelEx(&cfg, empty_k, a, out); }));
  cudaStreamSynchronize(s);
  cudaGraph_t g;
  cudaGraphExec_t ge;
  cudaStream_t cs;
  cudaStreamCreateWithFlags(&cs, cudaStreamNonBlocking);
  cfg.stream = cs;
  cudaStreamBeginCapture(cs, cudaStreamCaptureModeThreadLocal);
  cudaLaunchKernelEx(&cfg, empty_k, a, out);
  cudaStreamEndCapture(cs, &g);
  cudaGraphInstantiate(&ge, g, 0);
  size_t n = 1;
  cudaGraphNode_t node;
  cudaGraphGetNodes(g, &node, &n);
  cudaKernelNodeParams kp;
  cudaGraphKernelNodeGetParams(node, &kp);
  printf("graph     %.2f us\n", med_us([&] { cudaGraphLaunch(ge, s); }));
  cudaStreamSynchronize(s);
  long long k = 0;
  printf("graph+set %.2f us\n", med_us([&] {
    a.x[1] = ++k;
    void* args[] = {&a, &out};
    kp.kernelParams = args;
    cudaGraphExecKernelNodeSetParams(ge, node, &kp);
    cudaGraphLaunch(ge, s);
  }));
  cudaStreamSynchronize(s);
  // device span of a launch on an idle stream
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  std::vector<float> sp;
  for (int i = 0; i < 200; ++i) {
    cudaEventRecord(e0, s);
    cudaGraphLaunch(ge, s);
    cudaEventRecord(e1, s);
    cudaEventSynchronize(e1);
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    sp.push_back(ms * 1e3f);
  }
  std::sort(sp.begin(), sp.end());
  printf("graph span %.2f us (idle stream)\n", sp[sp.size() / 2]);
  sp.clear();
  cfg.stream = s;
  for (int i = 0; i < 200; ++i) {
    cudaEventRecord(e0, s);
    cudaLaunchKernelEx(&cfg, empty_k, a, out);
    cudaEventRecord(e1, s);
    cudaEventSynchronize(e1);
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    sp.push_back(ms * 1e3f);
  }
  std::sort(sp.begin(), sp.end());
  printf("cluster span %.2f us (idle stream)\n", sp[sp.size() / 2]);
  printf("err %s\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}
