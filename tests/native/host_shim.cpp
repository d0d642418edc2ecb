// Host build of the device headers (TEST INFRASTRUCTURE): lets the CPU suite
// check the exact device arithmetic (glibc tanh restatement, fold shapes)
// against the host libm and the oracle without a GPU.
#include "../../paper_2208_14228_b200/csrc/bt_libm.cuh"

extern "C" {
double shim_tanh(double x) { return bt::glibc_tanh(x); }
double shim_tanh_simt(double x) { return bt::glibc_tanh_simt(x); }
double shim_expm1(double x) { return bt::glibc_expm1_fma(x); }
double shim_streamfold(const double* v, int n, int fanin) {
  bt::StreamFold<double, 24> f;
  f.init(fanin);
  for (int i = 0; i < n; ++i) f.push(v[i]);
  return f.finish();
}
float shim_streamfold_f32(const float* v, int n, int fanin) {
  bt::StreamFold<float, 24> f;
  f.init(fanin);
  for (int i = 0; i < n; ++i) f.push(v[i]);
  return f.finish();
}
#define TL(N)                                                              \
  double shim_tree2_##N(const double* v) {                                 \
    double b[N];                                                           \
    for (int i = 0; i < N; ++i) b[i] = v[i];                               \
    return bt::TreeLevel<N, 2>::run(b);                                    \
  }                                                                        \
  double shim_seq_##N(const double* v) {                                   \
    double b[N];                                                           \
    for (int i = 0; i < N; ++i) b[i] = v[i];                               \
    return bt::TreeLevel<N, 0>::run(b);                                    \
  }
TL(1) TL(2) TL(4) TL(8) TL(16) TL(32) TL(64) TL(5) TL(12)
}
