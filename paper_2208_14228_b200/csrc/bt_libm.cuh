// bt_libm.cuh -- binary64 tanh that is bit-identical to the reference's.
//
// The reference evaluates `math.tanh` (model.py:148), i.e. the host libm.  On
// the build and GPU images that is glibc 2.39 on x86-64: `tanh` is the generic
// fdlibm-derived routine (sysdeps/ieee754/dbl-64/s_tanh.c) and it calls
// `expm1`, an IFUNC whose FMA variant (s_expm1.c compiled with -mfma) is
// selected on every FMA-capable host.  This file restates exactly that
// evaluation -- including WHICH multiply-adds glibc's compiled code fuses
// (read off `objdump -d libm.so.6`: vfmadd/vfnmadd/vfmsub at the polynomial,
// the t=3-r1*hfx / 6-x*t terms, the final corrections) -- with __fma_rn where
// glibc fused and explicit round-to-nearest mul/add everywhere else.
//
// Verified bit-exact against the host libm on 2e7 inputs (tests/test_libm_port.py
// runs the same source compiled for the host; tests/test_gpu_parity.py runs it
// on the B200).  The algorithm is the public fdlibm/glibc one; the constants
// are fdlibm's published ones.
#pragma once

#include "bt_common.cuh"

namespace bt {

BT_HD uint32_t hi_word(double x) { return (uint32_t)(d2u(x) >> 32); }
BT_HD uint32_t lo_word(double x) { return (uint32_t)d2u(x); }
BT_HD double with_hi(double x, uint32_t h) { return u2d(((uint64_t)h << 32) | (d2u(x) & 0xffffffffull)); }

BT_HD double glibc_expm1_fma(double x) {
  const double ln2_hi = 6.93147180369123816490e-01, ln2_lo = 1.90821492927058770002e-10,
               invln2 = 1.44269504088896338700e+00;
  const double Q1 = -3.33333333333331316428e-02, Q2 = 1.58730158725481460165e-03,
               Q3 = -7.93650757867487942473e-05, Q4 = 4.00821782732936239552e-06,
               Q5 = -2.01099218183624371326e-07;
  uint32_t hx = hi_word(x);
  const uint32_t xsb = hx & 0x80000000u;
  hx &= 0x7fffffffu;
  double hi, lo, c = 0.0, t, e, y;
  int k;
  if (hx >= 0x4043687Au) {    // |x| >= 56 ln2
    if (hx >= 0x40862E42u) {  // |x| >= 709.78
      if (hx >= 0x7ff00000u) {
        if (((hx & 0xfffffu) | lo_word(x)) != 0) return dadd(x, x);  // NaN
        return xsb == 0 ? x : -1.0;
      }
      if (x > 7.09782712893383973096e+02) return dmul(1e300, 1e300);  // overflow
    }
    if (xsb) return dsub(1e-300, 1.0);  // -1 with inexact
  }
  if (hx > 0x3fd62e42u) {  // |x| > 0.5 ln2
    if (hx < 0x3FF0A2B2u) {  // and |x| < 1.5 ln2
      if (!xsb) { hi = dsub(x, ln2_hi); lo = ln2_lo; k = 1; }
      else { hi = dadd(x, ln2_hi); lo = -ln2_lo; k = -1; }
    } else {
      k = (int)dadd(dmul(invln2, x), xsb == 0 ? 0.5 : -0.5);  // not fused in glibc's code
      t = (double)k;
      hi = dfma(-t, ln2_hi, x);  // fused (exact either way: t*ln2_hi is exact)
      lo = dmul(t, ln2_lo);
    }
    x = dsub(hi, lo);
    c = dsub(dsub(hi, x), lo);
  } else if (hx < 0x3c900000u) {  // |x| < 2^-54
    return x;
  } else {
    k = 0;
  }
  const double hfx = dmul(0.5, x);
  const double hxs = dmul(x, hfx);
  const double R1 = dfma(hxs, Q1, 1.0);
  const double h2 = dmul(hxs, hxs);
  const double R2 = dfma(hxs, Q3, Q2);
  const double h4 = dmul(h2, h2);
  const double R3 = dfma(hxs, Q5, Q4);
  const double r1 = dfma(h4, R3, dfma(h2, R2, R1));
  t = dfma(-r1, hfx, 3.0);
  e = dmul(hxs, ddiv(dsub(r1, t), dfma(-x, t, 6.0)));
  if (k == 0) return dsub(x, dfma(x, e, -hxs));
  e = dfma(dsub(e, c), x, -c);
  e = dsub(e, hxs);
  if (k == -1) return dfma(0.5, dsub(x, e), -0.5);
  if (k == 1) {
    if (x < -0.25) return dmul(-2.0, dsub(e, dadd(x, 0.5)));
    return dfma(dsub(x, e), 2.0, 1.0);
  }
  if (k <= -2 || k > 56) {
    y = dsub(1.0, dsub(e, x));
    y = with_hi(y, hi_word(y) + ((uint32_t)k << 20));
    return dsub(y, 1.0);
  }
  if (k < 20) {
    t = u2d((uint64_t)(0x3ff00000u - (0x200000u >> k)) << 32);
    y = dsub(t, dsub(e, x));
    y = with_hi(y, hi_word(y) + ((uint32_t)k << 20));
  } else {
    t = u2d((uint64_t)((uint32_t)(0x3ff - k) << 20) << 32);
    y = dsub(x, dadd(e, t));
    y = dadd(y, 1.0);
    y = with_hi(y, hi_word(y) + ((uint32_t)k << 20));
  }
  return y;
}

// glibc s_tanh.c (generic, not an IFUNC: no fused ops).
BT_HD double glibc_tanh(double x) {
  const uint32_t jx = hi_word(x), ix = jx & 0x7fffffffu, lx = lo_word(x);
  double t, z;
  if (ix >= 0x7ff00000u) {  // inf or NaN
    if (!(jx >> 31)) return dadd(ddiv(1.0, x), 1.0);
    return dsub(ddiv(1.0, x), 1.0);
  }
  if (ix < 0x40360000u) {  // |x| < 22
    if ((ix | lx) == 0) return x;          // +-0
    if (ix < 0x3c800000u) return dmul(x, dadd(1.0, x));  // |x| < 2^-55
    const double ax = fabs(x);
    if (ix >= 0x3ff00000u) {  // |x| >= 1
      t = glibc_expm1_fma(dadd(ax, ax));
      z = dsub(1.0, ddiv(2.0, dadd(t, 2.0)));
    } else {
      t = glibc_expm1_fma(dmul(-2.0, ax));
      z = ddiv(-t, dadd(t, 2.0));
    }
  } else {
    z = dsub(1.0, 1e-300);  // |x| >= 22 -> +-1
  }
  return (jx >> 31) ? -z : z;
}

// ---------------------------------------------------------------------------
// Branch-free restatement for SIMT execution.  glibc's control flow diverges
// across a warp (|x| >= 1 or not in tanh; k = 0, +-1, general, < 20, > 56 in
// expm1), serialising up to ~6 paths.  The version below evaluates the
// common polynomial once and every cheap reconstruction formula, then selects
// -- each lane performs exactly the operations glibc performs for its input:
//  * argument reduction: for k = +-1 glibc computes hi = x -+ ln2_hi,
//    lo = +-ln2_lo; fma(-t, ln2_hi, x) and t*ln2_lo with t = +-1 are the same
//    single roundings, and with t = 0 they return x and 0 exactly (x' = x);
//  * tanh: num/(t+2) with num = 2 (|x| >= 1) or -t, then 1-q or q.
// Only tanh's rare special inputs (NaN/inf, +-0, |x| < 2^-55, |x| >= 22) take
// the scalar glibc path.  Inside tanh, expm1 sees x in [-2, -2^-54) u [2, 44),
// so none of expm1's special branches can trigger there.
BT_HD double glibc_expm1_fma_tanh_domain(double x) {
  const double ln2_hi = 6.93147180369123816490e-01, ln2_lo = 1.90821492927058770002e-10,
               invln2 = 1.44269504088896338700e+00;
  const double Q1 = -3.33333333333331316428e-02, Q2 = 1.58730158725481460165e-03,
               Q3 = -7.93650757867487942473e-05, Q4 = 4.00821782732936239552e-06,
               Q5 = -2.01099218183624371326e-07;
  const uint32_t hx = hi_word(x) & 0x7fffffffu;
  const bool neg = (hi_word(x) >> 31) != 0;
  const double kgd = dtrunc(dadd(dmul(invln2, x), neg ? -0.5 : 0.5));  // (int) truncation, kept in binary64
  const double tk = hx <= 0x3fd62e42u ? 0.0 : (hx < 0x3FF0A2B2u ? (neg ? -1.0 : 1.0) : kgd);
  const int k = (int)tk;  // exact (|k| <= 64 in the tanh domain); off the critical path
  const double hi = dfma(-tk, ln2_hi, x);
  const double lo = dmul(tk, ln2_lo);
  const double xr = dsub(hi, lo);
  const double c = dsub(dsub(hi, xr), lo);
  const double hfx = dmul(0.5, xr);
  const double hxs = dmul(xr, hfx);
  const double R1 = dfma(hxs, Q1, 1.0);
  const double h2 = dmul(hxs, hxs);
  const double R2 = dfma(hxs, Q3, Q2);
  const double h4 = dmul(h2, h2);
  const double R3 = dfma(hxs, Q5, Q4);
  const double r1 = dfma(h4, R3, dfma(h2, R2, R1));
  const double t = dfma(-r1, hfx, 3.0);
  const double e = dmul(hxs, ddiv_normal(dsub(r1, t), dfma(-xr, t, 6.0)));  // num ~ -2, den ~ 6
  const double res0 = dsub(xr, dfma(xr, e, -hxs));           // k == 0
  const double e2 = dsub(dfma(dsub(e, c), xr, -c), hxs);
  const double resm1 = dfma(0.5, dsub(xr, e2), -0.5);        // k == -1
  const double res1 = xr < -0.25 ? dmul(-2.0, dsub(e2, dadd(xr, 0.5))) : dfma(dsub(xr, e2), 2.0, 1.0);
  const uint32_t kshift = (uint32_t)k << 20;
  const double yb = dsub(1.0, dsub(e2, xr));                 // k <= -2 || k > 56
  const double resb = dsub(with_hi(yb, hi_word(yb) + kshift), 1.0);
  const int kl = k < 0 ? 0 : (k > 31 ? 31 : k);              // 2 <= k < 20 (clamped: no UB shifts)
  const double tl = u2d((uint64_t)(0x3ff00000u - (0x200000u >> kl)) << 32);
  const double yl = dsub(tl, dsub(e2, xr));
  const double resl = with_hi(yl, hi_word(yl) + kshift);
  const int kh = k < 0 ? 0 : (k > 0x3ff ? 0x3ff : k);        // 20 <= k <= 56
  const double th = u2d((uint64_t)((uint32_t)(0x3ff - kh) << 20) << 32);
  const double yh = dadd(dsub(xr, dadd(e2, th)), 1.0);
  const double resh = with_hi(yh, hi_word(yh) + kshift);
  double r = resh;
  r = k < 20 ? resl : r;
  r = (k <= -2 || k > 56) ? resb : r;
  r = k == 1 ? res1 : r;
  r = k == -1 ? resm1 : r;
  r = k == 0 ? res0 : r;
  return r;
}

BT_HD double glibc_tanh_simt(double x) {
  const uint32_t jx = hi_word(x), ix = jx & 0x7fffffffu, lx = lo_word(x);
  const double ax = fabs(x);
  const bool big = ix >= 0x3ff00000u;  // |x| >= 1
  const double t = glibc_expm1_fma_tanh_domain(big ? dadd(ax, ax) : dmul(-2.0, ax));
  const double q = ddiv_normal(big ? 2.0 : -t, dadd(t, 2.0));
  const double z = big ? dsub(1.0, q) : q;
  double r = (jx >> 31) ? -z : z;
  // glibc's early returns, as selects (no branch; the general path above is
  // harmless garbage for these inputs and is discarded):
  //   |x| >= 22 or inf: +-(1 - 1e-300) = +-1 (inf: 1/x +- 1 = +-1)
  //   |x| < 2^-55, +-0 included: x * (1 + x)  (glibc returns x for +-0: same bits)
  //   NaN: a NaN (binary64 NaN results are canonical on the GPU either way)
  r = ix >= 0x40360000u ? ((jx >> 31) ? -1.0 : 1.0) : r;
  r = ix < 0x3c800000u ? dmul(x, dadd(1.0, x)) : r;
  r = (ix > 0x7ff00000u || (ix == 0x7ff00000u && lx != 0)) ? dadd(x, x) : r;
  return r;
}

}  // namespace bt
