// omb_pow.cuh -- glibc's double pow, restated for the device (and the host,
// for the CPU emulation harness), so tau (the dual-energy entropy tracer) is
// bit-identical to the reference, whose numpy/Cython path calls glibc ``pow``
// (reference: _kernels/reference.py:39, hydro/eos.py:50-61).
//
// Algorithm: glibc 2.28+ pow (sysdeps/ieee754/dbl-64/e_pow.c, by Szabolcs
// Nagy): log(x) in double-double from a 128-entry (invc, logc, logctail)
// table and a degree-8 polynomial, y*log(x) split exactly, exp from a
// 128-entry 2^(k/128) table and a degree-5 polynomial, result scale*(1+tmp).
// x86-64 glibc selects its FMA build (__pow_fma) on CPUs with FMA+AVX2, and
// gcc contracted its a*b+c expressions; the contraction pattern below was read
// off this image's libm.so.6 (objdump of __pow_fma) and every fma() here is
// one of its vfmadd/vfmsub instructions -- nothing else may contract, so this
// file is compiled with -fmad=false (device) / -ffp-contract=off (host).
// Tables: omb_pow_tables.cuh, extracted from the same libm by
// gen_glibc_pow_tables.py.  Checked bitwise against the host's pow on 2^24
// random pairs plus edge cases (tests/test_pow.py on the CPU, and the device
// copy in tests/test_gpu_parity.py::test_device_pow_is_glibc).
#pragma once
#include <math.h>
#include <stdint.h>
#include <string.h>

#ifndef OMB_HD
#ifdef __CUDACC__
#define OMB_HD __host__ __device__ __forceinline__
#else
#define OMB_HD inline
#endif
#endif

namespace omb {
namespace glibc_pow_host {
#define OMB_POW_CONST static const
#include "omb_pow_tables.cuh"
#undef OMB_POW_CONST
}  // namespace glibc_pow_host
#ifdef __CUDACC__
namespace glibc_pow_dev {
// global memory through the read-only path: the table index differs per lane
#define OMB_POW_CONST static __device__ const
#include "omb_pow_tables.cuh"
#undef OMB_POW_CONST
}  // namespace glibc_pow_dev
#endif

namespace gp {

#ifdef __CUDA_ARCH__
#define OMB_PT(name) glibc_pow_dev::name
OMB_HD double ld(const double* p) { return __ldg(p); }
OMB_HD unsigned long long ldu(const unsigned long long* p) { return __ldg(p); }
OMB_HD uint64_t bits(double x) { return (uint64_t)__double_as_longlong(x); }
OMB_HD double dbl(uint64_t i) { return __longlong_as_double((long long)i); }
#else
#define OMB_PT(name) glibc_pow_host::name
OMB_HD double ld(const double* p) { return *p; }
OMB_HD unsigned long long ldu(const unsigned long long* p) { return *p; }
OMB_HD uint64_t bits(double x) {
  uint64_t i;
  memcpy(&i, &x, 8);
  return i;
}
OMB_HD double dbl(uint64_t i) {
  double x;
  memcpy(&x, &i, 8);
  return x;
}
#endif

constexpr uint64_t OFF = 0x3fe6955500000000ull;
constexpr uint64_t SIGN_BIAS = 0x800ull << 7;

OMB_HD uint32_t top12(double x) { return (uint32_t)(bits(x) >> 52); }
OMB_HD bool zeroinfnan(uint64_t i) { return 2 * i - 1 >= 2 * 0x7ff0000000000000ull - 1; }
// 0: not an integer, 1: odd integer, 2: even integer
OMB_HD int checkint(uint64_t iy) {
  int e = (int)(iy >> 52 & 0x7ff);
  if (e < 0x3ff) return 0;
  if (e > 0x3ff + 52) return 2;
  if (iy & ((1ull << (0x3ff + 52 - e)) - 1)) return 0;
  if (iy & (1ull << (0x3ff + 52 - e))) return 1;
  return 2;
}

// log(x) = hi + tail for normal positive x bits ix (e_pow.c log_inline)
OMB_HD double log_inline(uint64_t ix, double& tail) {
  const double* H = OMB_PT(kLogHead);
  uint64_t tmp = ix - OFF;
  int i = (int)((tmp >> 45) % 128);
  int k = (int)((int64_t)tmp >> 52);
  uint64_t iz = ix - (tmp & (0xfffull << 52));
  double z = dbl(iz);
  double kd = (double)k;
  const double* T = OMB_PT(kLogTab)[i];
  double invc = ld(T), logc = ld(T + 1), logctail = ld(T + 2);
  double r = fma(z, invc, -1.0);
  double t1 = fma(kd, ld(H + 0), logc);      // k*Ln2hi + logc
  double t2 = t1 + r;
  double lo1 = fma(kd, ld(H + 1), logctail);  // k*Ln2lo + logctail
  double lo2 = t1 - t2 + r;
  double ar = ld(H + 2) * r;  // A[0] = -0.5
  double ar2 = r * ar;
  double ar3 = r * ar2;
  double hi = t2 + ar2;
  double lo3 = fma(ar, r, -ar2);
  double lo4 = t2 - hi + ar2;
  // p = ar3 * (A1 + r A2 + ar2 (A3 + r A4 + ar2 (A5 + r A6))), the last product fused into lo
  double q12 = fma(r, ld(H + 4), ld(H + 3));
  double q34 = fma(r, ld(H + 6), ld(H + 5));
  double q56 = fma(r, ld(H + 8), ld(H + 7));
  double q = fma(ar2, fma(ar2, q56, q34), q12);
  double lo = fma(ar3, q, ((lo1 + lo2) + lo3) + lo4);
  double y = hi + lo;
  tail = hi - y + lo;
  return y;
}

// e_exp.c specialcase: |k| large, the scale exponent needs adjusting
OMB_HD double exp_special(double tmp, uint64_t sbits, uint64_t ki) {
  if ((ki & 0x80000000) == 0) {
    sbits -= 1009ull << 52;
    double scale = dbl(sbits);
    return 0x1p1009 * fma(scale, tmp, scale);
  }
  sbits += 1022ull << 52;
  double scale = dbl(sbits);
  double st = scale * tmp;
  double y = scale + st;
  if (fabs(y) < 1.0) {
    double one = y < 0.0 ? -1.0 : 1.0;
    double lo = scale - y + st;
    double hi = y + one;
    lo = one - hi + y + lo;
    y = (lo + hi) - one;
    if (y == 0) y = dbl(sbits & 0x8000000000000000ull);
  }
  return y * 0x1p-1022;
}

// exp(x + xtail) with the sign bias of pow (e_pow.c exp_inline)
OMB_HD double exp_inline(double x, double xtail, uint64_t sign_bias) {
  const double* E = OMB_PT(kExpHead);
  uint32_t abstop = top12(x) & 0x7ff;
  if (abstop - top12(0x1p-54) >= top12(512.0) - top12(0x1p-54)) {
    if (abstop - top12(0x1p-54) >= 0x80000000u) {
      double one = 1.0 + x;
      return sign_bias ? -one : one;
    }
    if (abstop >= top12(1024.0)) {
      // __math_uflow / __math_oflow: +-0 or +-inf
      double r = (bits(x) >> 63) ? 0.0 : INFINITY;
      return sign_bias ? -r : r;
    }
    abstop = 0;  // large |x|: handled by exp_special
  }
  double kd = fma(x, ld(E + 0), ld(E + 1));  // InvLn2N * x + Shift
  uint64_t ki = bits(kd);
  kd -= ld(E + 1);
  double r = fma(kd, ld(E + 2), x);  // + kd * NegLn2hiN
  r = fma(kd, ld(E + 3), r);         // + kd * NegLn2loN
  r = xtail + r;
  uint64_t idx = 2 * (ki % 128);
  uint64_t top = (ki + sign_bias) << 45;
  double tail = dbl(ldu(OMB_PT(kExpTab) + idx));
  uint64_t sbits = ldu(OMB_PT(kExpTab) + idx + 1) + top;
  double r2 = r * r;
  double c23 = fma(r, ld(E + 5), ld(E + 4));
  double c45 = fma(r, ld(E + 7), ld(E + 6));
  double tmp = fma(r2 * r2, c45, fma(r2, c23, tail + r));
  if (abstop == 0) return exp_special(tmp, sbits, ki);
  double scale = dbl(sbits);
  return fma(scale, tmp, scale);
}

}  // namespace gp

// pow(x, y) bit-identical to glibc's (x86-64 FMA build)
OMB_HD double pow_glibc(double x, double y) {
  using namespace gp;
  uint64_t ix = bits(x), iy = bits(y);
  uint32_t topx = (uint32_t)(ix >> 52), topy = (uint32_t)(iy >> 52);
  uint64_t sign_bias = 0;
  if (topx - 0x001 >= 0x7ff - 0x001 || (topy & 0x7ff) - 0x3be >= 0x43e - 0x3be) {
    if (zeroinfnan(iy)) {
      if (2 * iy == 0) return 1.0;
      if (ix == 0x3ff0000000000000ull) return 1.0;
      if (2 * ix > 2 * 0x7ff0000000000000ull || 2 * iy > 2 * 0x7ff0000000000000ull) return x + y;
      if (2 * ix == 2 * 0x3ff0000000000000ull) return 1.0;
      if ((2 * ix < 2 * 0x3ff0000000000000ull) == !(iy >> 63)) return 0.0;
      return y * y;
    }
    if (zeroinfnan(ix)) {
      double x2 = x * x;
      if ((ix >> 63) && checkint(iy) == 1) x2 = -x2;
      return (iy >> 63) ? 1.0 / x2 : x2;
    }
    if (ix >> 63) {  // finite x < 0
      int yint = checkint(iy);
      if (yint == 0) return (x - x) / (x - x);  // invalid: NaN
      if (yint == 1) sign_bias = SIGN_BIAS;
      ix &= 0x7fffffffffffffffull;
      topx &= 0x7ff;
    }
    if ((topy & 0x7ff) - 0x3be >= 0x43e - 0x3be) {
      if (ix == 0x3ff0000000000000ull) return 1.0;
      if ((topy & 0x7ff) < 0x3be) return ix > 0x3ff0000000000000ull ? 1.0 + y : 1.0 - y;
      return ((ix > 0x3ff0000000000000ull) == (topy < 0x800)) ? INFINITY : 0.0;
    }
    if (topx == 0) {  // subnormal x: normalise
      ix = bits(x * 0x1p52);
      ix &= 0x7fffffffffffffffull;
      ix -= 52ull << 52;
    }
  }
  double lo;
  double hi = log_inline(ix, lo);
  double ehi = y * hi;
  double elo = fma(y, lo, fma(y, hi, -ehi));
  return exp_inline(ehi, elo, sign_bias);
}

}  // namespace omb
