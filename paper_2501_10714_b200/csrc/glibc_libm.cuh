// glibc_libm.cuh — bit-exact restatement of the host libm routines the
// reference's noisy gate calls, for host and device (sm_100a) code.
//
// The reference computes its noise as n = sqrt(-2 log u1) * cos(2 pi u2) and
// its softplus as log1p(exp(z)) (proj/src/workload.cpp:91-101), and its
// softmax / sigmoid weights with exp (123-133, 198). Those four libm
// functions are not correctly rounded, so a device that uses CUDA's own
// log / cos / exp / log1p can differ from the reference by an ulp — enough to
// flip a near-tie in the top-k. glibc 2.39 on an x86-64 host with FMA and
// AVX2 (the image's; glibc selects these variants by ifunc) runs
// __log_fma, __exp_fma, __log1p_fma and __cos_fma: the ARM optimized-routines
// log and exp, fdlibm's log1p and IBM's accurate sin/cos, compiled with
// fused multiply-adds. The functions below restate those instruction
// sequences operation by operation — every multiply, add and fused
// multiply-add where the FMA build has one, in the same order — over the
// constants and tables read out of that libm (glibc_libm_data.h, generated
// by tools/extract_glibc_libm.py). IEEE-754 double operations with
// round-to-nearest are deterministic, so the results carry the same bits as
// the host's libm; tests/test_glibc_libm.py checks that on the host against
// the live libm (every branch, 10^7+ random arguments per function) and
// tests/test_noise_exact_gpu.py on the device.
//
// Only finite arguments are in the gate's domain (u1, u2 in (0, 1), any
// finite z); the special-value paths (NaN, infinities, overflow) follow the
// same results without raising errno / FP flags.
#pragma once

#include <cstdint>
#include <cstring>

// nvcc: device functions over per-module tables; a host compiler (the CPU
// check, tests/test_glibc_libm.py): plain inline functions
#if defined(__CUDACC__)
#define GL_HD __device__ __forceinline__
#define GL_TABLE static __device__ const
#else
#include <cmath>
#define GL_HD inline
#define GL_TABLE inline const
#endif
#define GL_CONST constexpr

#include "glibc_libm_data.h"

namespace fsmoe_libm {

// ---- exact IEEE operations (no contraction, no reassociation) -------------
#if defined(__CUDACC__)
GL_HD double fma_(double a, double b, double c) { return __fma_rn(a, b, c); }
GL_HD double mul_(double a, double b) { return __dmul_rn(a, b); }
GL_HD double add_(double a, double b) { return __dadd_rn(a, b); }
GL_HD double sub_(double a, double b) { return __dsub_rn(a, b); }
GL_HD double div_(double a, double b) { return __ddiv_rn(a, b); }
GL_HD double sqrt_(double a) { return __dsqrt_rn(a); }
GL_HD double bits2d(uint64_t u) { return __longlong_as_double(static_cast<long long>(u)); }
GL_HD uint64_t d2bits(double d) { return static_cast<uint64_t>(__double_as_longlong(d)); }
#else
// host: the translation unit must be built without FP contraction
// (-ffp-contract=off); std::fma is the IEEE fused operation
GL_HD double fma_(double a, double b, double c) { return std::fma(a, b, c); }
GL_HD double mul_(double a, double b) {
  volatile double r = a * b;
  return r;
}
GL_HD double add_(double a, double b) {
  volatile double r = a + b;
  return r;
}
GL_HD double sub_(double a, double b) {
  volatile double r = a - b;
  return r;
}
GL_HD double div_(double a, double b) { return a / b; }
GL_HD double sqrt_(double a) { return std::sqrt(a); }
GL_HD double bits2d(uint64_t u) {
  double d;
  std::memcpy(&d, &u, 8);
  return d;
}
GL_HD uint64_t d2bits(double d) {
  uint64_t u;
  std::memcpy(&u, &d, 8);
  return u;
}
#endif
GL_HD double K(uint64_t u) { return bits2d(u); }
GL_HD double fnma_(double a, double b, double c) { return fma_(-a, b, c); }  // c - a*b, one rounding
GL_HD double fms_(double a, double b, double c) { return fma_(a, b, -c); }   // a*b - c, one rounding
GL_HD double absd(double x) { return bits2d(d2bits(x) & 0x7fffffffffffffffULL); }
GL_HD double negd(double x) { return bits2d(d2bits(x) ^ 0x8000000000000000ULL); }
GL_HD double copysignd(double mag, double sgn) {
  return bits2d((d2bits(mag) & 0x7fffffffffffffffULL) | (d2bits(sgn) & 0x8000000000000000ULL));
}
GL_HD double tab(const uint64_t* t, int i) { return bits2d(t[i]); }

// ---------------------------------------------------------------- log ------
// __log_fma (glibc 2.39 sysdeps/ieee754/dbl-64/e_log.c, optimized-routines).
GL_HD double gl_log(double x) {
  uint64_t ix = d2bits(x);
  // |x - 1| small: its own polynomial (LO = 1 - 0x1p-4, HI = 1 + 0x1.09p-4)
  if (ix - 0x3fee000000000000ULL < 0x0003090000000000ULL) {
    if (ix == 0x3ff0000000000000ULL) return 0.0;
    const double r = sub_(x, K(ONE));
    double p012 = fma_(r, K(LOG_B2), K(LOG_B1));
    double p345 = fma_(r, K(LOG_B5), K(LOG_B4));
    double p78 = fma_(r, K(LOG_B8), K(LOG_B7));
    const double r2 = mul_(r, r);
    p012 = fma_(r2, K(LOG_B3), p012);
    p345 = fma_(r2, K(LOG_B6), p345);
    const double r3 = mul_(r, r2);
    double p = fma_(r2, K(LOG_B9), p78);
    p = fma_(r3, K(LOG_B10), p);
    p = fma_(p, r3, p345);
    p = fma_(p, r3, p012);
    const double t = fma_(r, K(TWO27), r);       // r + r*2^27
    const double rhi = fnma_(K(TWO27), r, t);    // (r + w) - w
    const double rhi2 = mul_(rhi, rhi);
    const double rlo = sub_(r, rhi);
    const double hi = fma_(rhi2, K(LOG_B0), r);  // r + rhi^2 * B0
    const double d = sub_(r, hi);
    const double rr = add_(r, rhi);
    double lo = fma_(rhi2, K(LOG_B0), d);        // r - hi + w
    lo = fma_(mul_(K(LOG_B0), rlo), rr, lo);     // += B0 * rlo * (rhi + r)
    const double y = fma_(p, r3, lo);
    return add_(hi, y);
  }
  const uint64_t top = ix >> 48;
  if (top - 0x0010ULL >= 0x7ff0ULL - 0x0010ULL) {
    // zero, negative, subnormal, inf or NaN
    if ((ix << 1) == 0) return negd(bits2d(0x7ff0000000000000ULL));  // -inf
    if (ix == 0x7ff0000000000000ULL) return x;                         // +inf
    if ((top & 0x8000) || (top & 0x7ff0) == 0x7ff0) return bits2d(0x7ff8000000000000ULL);  // NaN
    // subnormal: scale into the normal range
    ix = d2bits(mul_(x, K(TWO52))) - (52ULL << 52);
  }
  const uint64_t tmp = ix - 0x3fe6000000000000ULL;
  const int i = static_cast<int>((tmp >> 45) & 0x7f);
  const int k = static_cast<int>(static_cast<int64_t>(tmp) >> 52);
  const uint64_t iz = ix - (tmp & 0xfff0000000000000ULL);
  const double invc = tab(LOG_TAB, 2 * i), logc = tab(LOG_TAB, 2 * i + 1);
  const double z = bits2d(iz);
  const double kd = static_cast<double>(k);
  const double w = fma_(kd, K(LOG_LN2HI), logc);
  const double r = fma_(z, invc, K(MINUS_ONE));
  const double a21 = fma_(r, K(LOG_A2), K(LOG_A1));
  const double hi = add_(r, w);
  const double r2 = mul_(r, r);
  double lo = add_(sub_(w, hi), r);
  lo = fma_(kd, K(LOG_LN2LO), lo);
  const double rr2 = mul_(r, r2);
  const double a43 = fma_(r, K(LOG_A4), K(LOG_A3));
  lo = fma_(r2, K(LOG_A0), lo);
  const double q = fma_(a43, r2, a21);
  const double y = fma_(rr2, q, lo);
  return add_(y, hi);
}

// ---------------------------------------------------------------- exp ------
// __exp_fma (e_exp.c, optimized-routines; N = 128).
GL_HD double gl_exp_special(double tmp, uint64_t sbits, uint64_t ki) {
  if ((ki & 0x80000000ULL) == 0) {
    // k > 0: the exponent of scale might have overflowed by <= 460
    sbits -= 1009ULL << 52;
    const double scale = bits2d(sbits);
    return mul_(K(TWO_1009), fma_(scale, tmp, scale));
  }
  // k < 0: the result may be subnormal
  sbits += 1022ULL << 52;
  const double scale = bits2d(sbits);
  double y = add_(scale, mul_(tmp, scale));
  if (y < 1.0) {
    const double st = mul_(tmp, scale);
    const double hi = add_(y, K(ONE));
    double lo = add_(sub_(scale, y), st);
    double yy = add_(sub_(K(ONE), hi), y);
    yy = add_(yy, lo);
    yy = add_(yy, hi);
    y = sub_(yy, K(ONE));
    if (y == 0.0) y = 0.0;
  }
  return mul_(y, K(TWO_M1022));
}

GL_HD double gl_exp(double x) {
  const uint64_t ix = d2bits(x);
  uint32_t abstop = static_cast<uint32_t>((ix >> 52) & 0x7ff);
  if (abstop - 0x3c9u > 0x3eu) {
    if (static_cast<int32_t>(abstop - 0x3c9u) < 0) return add_(x, K(ONE));  // |x| < 2^-54
    if (abstop >= 0x409) {                                                    // |x| >= 1024
      if (ix == 0xfff0000000000000ULL) return 0.0;
      if (abstop == 0x7ff) return add_(x, K(ONE));
      return (ix >> 63) ? 0.0 : bits2d(0x7ff0000000000000ULL);
    }
    abstop = 0;  // large |x| < 1024: the scale needs special care
  }
  const double z = fma_(x, K(EXP_INVLN2N), K(EXP_SHIFT));  // kd + shift
  const uint64_t ki = d2bits(z);
  const double kd = sub_(z, K(EXP_SHIFT));
  double r = fma_(kd, K(EXP_NEGLN2HIN), x);
  r = fma_(kd, K(EXP_NEGLN2LON), r);
  const int idx = 2 * static_cast<int>(ki & 0x7f);
  const uint64_t top = ki << 45;
  const double c32 = fma_(r, K(EXP_C3), K(EXP_C2));
  const double tail_r = add_(r, tab(EXP_TAB, idx));
  const uint64_t sbits = EXP_TAB[idx + 1] + top;
  const double r2 = mul_(r, r);
  const double c54 = fma_(r, K(EXP_C5), K(EXP_C4));
  const double t = fma_(c32, r2, tail_r);
  const double tmp = fma_(mul_(r2, r2), c54, t);
  if (abstop == 0) return gl_exp_special(tmp, sbits, ki);
  const double scale = bits2d(sbits);
  return fma_(scale, tmp, scale);
}

// -------------------------------------------------------------- log1p ------
// __log1p_fma (s_log1p.c, fdlibm).
GL_HD int32_t hi_word(double x) { return static_cast<int32_t>(d2bits(x) >> 32); }
GL_HD double with_hi_word(double x, uint32_t hw) {
  return bits2d((d2bits(x) & 0xffffffffULL) | (static_cast<uint64_t>(hw) << 32));
}

GL_HD double gl_log1p(double x) {
  const int32_t hx = hi_word(x);
  int k = 0;
  int32_t hu = 0;
  double f = 0.0, c = 0.0, u = x;
  bool k0 = false;  // the fdlibm k = 0 case (f = x)
  if (hx <= 0x3fda8279) {
    const uint32_t ax = static_cast<uint32_t>(hx) & 0x7fffffffu;
    if (ax > 0x3fefffffu) {  // x <= -1
      if (x == -1.0) return negd(bits2d(0x7ff0000000000000ULL));
      return bits2d(0x7ff8000000000000ULL);
    }
    if (ax <= 0x3e1fffffu) {  // |x| < 2^-29
      if (ax > 0x3c8fffffu) return fnma_(mul_(x, x), K(HALF), x);
      return x;
    }
    if (static_cast<uint32_t>(hx) + 0x402d413cu > 0x402d413cu) {
      k0 = true;  // -0.2929 < x < 0.41422
      f = x;
      hu = hx;
    }
  } else if (hx > 0x7fefffff) {
    return add_(x, x);
  }
  if (!k0) {
    if (hx <= 0x433fffff) {
      u = add_(x, K(ONE));
      hu = hi_word(u);
      k = (hu >> 20) - 1023;
      c = k > 0 ? sub_(K(ONE), sub_(u, x)) : sub_(x, sub_(u, K(ONE)));
      c = div_(c, u);
    } else {
      k = (hx >> 20) - 1023;
      u = x;
      hu = hx;
      c = 0.0;
    }
    hu &= 0x000fffff;
    if (hu <= 0x6a09d) {
      u = with_hi_word(u, static_cast<uint32_t>(hu) | 0x3ff00000u);
    } else {
      k += 1;
      u = with_hi_word(u, static_cast<uint32_t>(hu) | 0x3fe00000u);
      hu = (0x00100000 - hu) >> 2;
    }
    f = sub_(u, K(ONE));
  }
  const double hfsq = mul_(mul_(f, K(HALF)), f);
  if (!k0 && hu == 0) {  // |f| < 2^-20
    if (f == 0.0) {
      if (k == 0) return 0.0;
      const double kd = static_cast<double>(k);
      return fma_(kd, K(L1P_LN2_HI), fma_(kd, K(L1P_LN2_LO), c));
    }
    const double R = mul_(fnma_(f, K(L1P_TWO3), K(ONE)), hfsq);
    if (k == 0) return sub_(f, R);
    const double kd = static_cast<double>(k);
    const double t = sub_(sub_(R, fma_(kd, K(L1P_LN2_LO), c)), f);
    return fms_(kd, K(L1P_LN2_HI), t);
  }
  const double s = div_(f, add_(f, K(TWO)));
  const double z = mul_(s, s);
  const double r2 = fma_(z, K(L1P_LP3), K(L1P_LP2));
  const double r3 = fma_(z, K(L1P_LP5), K(L1P_LP4));
  const double r4 = fma_(z, K(L1P_LP7), K(L1P_LP6));
  const double z2 = mul_(z, z);
  const double z4 = mul_(z2, z2);
  const double z6 = mul_(z2, z4);
  double R = fma_(z, K(L1P_LP1), mul_(z2, r2));
  R = fma_(z4, r3, R);
  R = fma_(z6, r4, R);
  const double sr = mul_(add_(R, hfsq), s);
  if (k == 0) return sub_(f, sub_(hfsq, sr));
  const double kd = static_cast<double>(k);
  double t = add_(fma_(kd, K(L1P_LN2_LO), c), sr);
  t = sub_(sub_(hfsq, t), f);
  return fms_(kd, K(L1P_LN2_HI), t);
}

// ---------------------------------------------------------------- cos ------
// __cos_fma (s_sin.c, IBM Accurate Mathematical Library).
GL_HD int sincos_index(double u) { return static_cast<int>(static_cast<uint32_t>(d2bits(u))) << 2; }

// do_cos(x, dx): cos(x + dx) by table lookup around |x|
GL_HD double gl_do_cos(double x, double dx) {
  if (x < 0) dx = negd(dx);
  const double ax = absd(x);
  const double u = add_(ax, K(BIG));
  const int k = sincos_index(u);
  const double xr = add_(sub_(ax, sub_(u, K(BIG))), dx);
  const double xx = mul_(xr, xr);
  const double ps = fma_(xx, K(SN5), K(SN3));
  const double s = fma_(mul_(xr, xx), ps, xr);
  double pc = fma_(xx, K(CS6), K(CS4));
  pc = fma_(xx, pc, K(HALF));
  const double c = mul_(xx, pc);
  const double sn = tab(SINCOS_TAB, k), ssn = tab(SINCOS_TAB, k + 1);
  const double cs = tab(SINCOS_TAB, k + 2), ccs = tab(SINCOS_TAB, k + 3);
  double cor = fnma_(s, ssn, ccs);
  cor = fnma_(c, cs, cor);
  cor = fnma_(s, sn, cor);
  return add_(cs, cor);
}

// TAYLOR_SIN(a*a, a, da)
GL_HD double gl_taylor_sin(double a, double da) {
  const double xx = mul_(a, a);
  double p = fma_(xx, K(TS5), K(TS4));
  p = fma_(xx, p, K(TS3));
  p = fma_(xx, p, K(TS2));
  p = fma_(xx, p, K(TS1));
  const double t = fma_(xx, fms_(p, a, mul_(da, K(HALF))), da);
  return add_(t, a);
}

// do_sin(a, da): sin(a + da)
GL_HD double gl_do_sin(double a, double da) {
  const double aa = absd(a);
  if (K(SIN_TAYLOR_LIMIT) > aa) return gl_taylor_sin(a, da);
  if (!(0.0 < a)) da = negd(da);
  const double u = add_(aa, K(BIG));
  const int k = sincos_index(u);
  const double x = sub_(aa, sub_(u, K(BIG)));
  const double xx = mul_(x, x);
  const double ps = fma_(xx, K(SN5), K(SN3));
  const double s = add_(x, fma_(mul_(x, xx), ps, da));
  double pc = fma_(xx, K(CS6), K(CS4));
  pc = fma_(xx, pc, K(HALF));
  const double c = fma_(x, da, mul_(xx, pc));
  const double sn = tab(SINCOS_TAB, k), ssn = tab(SINCOS_TAB, k + 1);
  const double cs = tab(SINCOS_TAB, k + 2), ccs = tab(SINCOS_TAB, k + 3);
  double cor = fma_(s, ccs, ssn);
  cor = fnma_(c, sn, cor);
  cor = fma_(s, cs, cor);
  return copysignd(add_(sn, cor), a);
}

GL_HD double gl_cos(double x) {
  const uint32_t k = static_cast<uint32_t>(hi_word(x)) & 0x7fffffffu;
  if (k < 0x3e400000u) return K(ONE);  // |x| < 2^-27
  if (k < 0x3feb6000u) return gl_do_cos(x, 0.0);
  if (k < 0x400368fdu) {  // 0.855469 < |x| < 2.426265: sin(pi/2 - |x|)
    const double y = sub_(K(HP0), absd(x));
    const double a = add_(y, K(HP1));
    const double da = add_(sub_(y, a), K(HP1));
    return gl_do_sin(a, da);
  }
  if (k < 0x419921fbu) {  // |x| < 105414350: reduce by pi/2 in 106 bits
    const double t = fma_(x, K(HPINV), K(TOINT));
    const double xn = sub_(t, K(TOINT));
    const int n = static_cast<int>(d2bits(t) & 3);
    double y = fnma_(xn, K(MP1), x);
    y = fnma_(xn, K(MP2), y);
    const double t2 = fnma_(xn, K(PP3), y);
    double db = fnma_(xn, K(PP3), sub_(y, t2));
    const double b = fnma_(xn, K(PP4), t2);
    db = add_(db, fnma_(xn, K(PP4), sub_(t2, b)));
    const int m = n + 1;
    const double r = (m & 1) ? gl_do_cos(b, db) : gl_do_sin(b, db);
    return (m & 2) ? negd(r) : r;
  }
  // |x| >= 105414350 (or inf / NaN): outside the gate's domain (2 pi u2 < 2 pi)
  return bits2d(0x7ff8000000000000ULL);
}

// ------------------------------------------------------------ composites --
// workload.cpp:90-95: one normal draw from two 53-bit uniforms
GL_HD double gl_normal(double u1, double u2) {
  return mul_(sqrt_(mul_(-2.0, gl_log(u1))),
              gl_cos(mul_(6.283185307179586476925286766559, u2)));
}
// workload.cpp:101: softplus(z) = log1p(exp(z))
GL_HD double gl_softplus(double z) { return gl_log1p(gl_exp(z)); }

}  // namespace fsmoe_libm
